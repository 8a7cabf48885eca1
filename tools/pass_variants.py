"""Experiment: timing-only variants of a mode-2 specialised pass source
(SVB_JIT_DUMP), to separate what a pass spends on FP64 work from what it
spends on shared-memory transitions and HBM.  The variants compute garbage;
only their run time means anything (tools/passrun.cu).

    python tools/pass_variants.py pass.cu noF|noT|noFT out.cu

noF   gate arithmetic removed (loads, transitions, barriers, stores kept)
noT   register-group transitions removed (shared-memory stores + reloads and
      their barriers); group 0's loads, the gates and the last group's HBM
      stores kept
noFT  both: the tile only travels HBM -> shared -> registers -> HBM
"""
import re
import sys


def split_groups(lines):
    """[(start, end)] line ranges of the '{ // group k' blocks (end exclusive,
    at the block's closing brace)."""
    starts = [i for i, ln in enumerate(lines) if re.match(r"\{ // group \d+", ln)]
    out = []
    for k, s in enumerate(starts):
        e = starts[k + 1] if k + 1 < len(starts) else len(lines)
        out.append((s, e))
    return out


def variant(src: str, kind: str) -> str:
    lines = src.split("\n")
    groups = split_groups(lines)
    drop = set()
    for gi, (s, e) in enumerate(groups):
        last = gi == len(groups) - 1
        # end of the loads: the 'v[31] = <load>' line (+ the last group's barrier and prefetch)
        ld_end = next(i for i in range(s, e) if re.match(r"v\[31\] = (\*reinterpret_cast|ldcs)", lines[i]))
        ld_start = next(i for i in range(s, e) if lines[i].startswith("unsigned a0"))
        gate_start = ld_end + 1
        while lines[gate_start].startswith("__syncthreads();") or "fill(" in lines[gate_start]:
            gate_start += 1
        # start of the store section
        st = next(i for i in range(gate_start, e) if lines[i].startswith("unsigned b0") or lines[i].startswith("unsigned s0"))
        if lines[st - 1].startswith("__syncthreads();") or lines[st - 1].startswith("__syncwarp();"):
            st -= 1
        if "F" in kind:
            drop.update(range(gate_start, st))
        if "T" in kind:
            if gi > 0:
                drop.update(range(ld_start, ld_end + 1))
            if not last:
                # the store section ends at the barrier before the group's closing brace
                end = max(i for i in range(st, e) if lines[i].startswith("__syncthreads();"))
                drop.update(range(st, end + 1))
    return "\n".join(ln for i, ln in enumerate(lines) if i not in drop)


if __name__ == "__main__":
    open(sys.argv[3], "w").write(variant(open(sys.argv[1]).read(), sys.argv[2]))
