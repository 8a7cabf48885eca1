"""Experiment: add warpgroup ping-pong to a tile-ring pass source (SVB_JIT_MODE=3
dump): the FP64 section of a register group runs only while the CTA's other
warpgroup is in its shared-memory / HBM section (named barriers 3 and 4 pass
a token back and forth), so the two tiles in flight on an SM alternate between
the FP64 pipe and the load/store pipes instead of colliding on either.

    python tools/pingpong_patch.py ring_pass.cu out.cu
"""
import re
import sys

PP = r"""
__device__ __forceinline__ void pp_wait(int wg) { asm volatile("bar.sync %0, 256;" :: "r"(3 + wg) : "memory"); }
__device__ __forceinline__ void pp_pass(int wg) { asm volatile("bar.arrive %0, 256;" :: "r"(4 - wg) : "memory"); }
"""


def patch(src: str) -> str:
    lines = src.split("\n")
    out = []
    ngroups = sum(1 for ln in lines if re.match(r"\{ // group \d+", ln))
    in_group = False
    waited = passed = False
    pending_wait_after_fill = False
    for i, ln in enumerate(lines):
        if ln.startswith("__constant__ double kc["):
            out.append(PP)
        if re.match(r"\{ // group \d+", ln):
            in_group, waited, passed = True, False, False
        if in_group and not passed and waited:
            nxt = lines[i + 1] if i + 1 < len(lines) else ""
            sync = ln.startswith("wg_sync(wg, 128);") or ln.startswith("__syncwarp();")
            if (sync and nxt.startswith("unsigned b0")) or ln.startswith("unsigned b0") or ln.startswith("unsigned s0 ="):
                out.append("pp_pass(wg);")
                passed = True
        if ln.startswith("if (tix >= ntiles) break;"):
            out.append("if (tix >= ntiles) { if (wg == 1 && blockIdx.x + (j - 1) * gridDim.x < ntiles) {"
                       + " pp_wait(wg); pp_pass(wg);" * ngroups + " } break; }")
            continue
        out.append(ln)
        if in_group and not waited:
            if re.match(r"v\[31\] = ", ln):
                nxt = lines[i + 1]
                if nxt.startswith("wg_sync(wg, 128);") and lines[i + 2].startswith("fill3("):
                    pending_wait_after_fill = True
                else:
                    out.append("pp_wait(wg);")
                    waited = True
            elif pending_wait_after_fill and ln.startswith("fill3("):
                out.append("pp_wait(wg);")
                waited = True
                pending_wait_after_fill = False
        if ln.startswith("if (wg == 0) { fill3(0, 0);"):
            out.append("if (wg == 1) pp_pass(wg);")
    # the loop's closing brace is the second-to-last '}' line; WG0 consumes the
    # last token so no arrival is left pending at exit
    k = len(out) - 1
    while not out[k].startswith("}"):
        k -= 1
    out.insert(k, "if (wg == 0) pp_wait(wg);")
    s = "\n".join(out)
    assert s.count("pp_wait(wg);") >= ngroups and s.count("pp_pass(wg);") >= ngroups, (ngroups, s.count("pp_wait"))
    return s


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))
