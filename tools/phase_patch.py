"""Experiment: clock64() stamps at the phase boundaries of a mode-2 pass
source; per-warp cycle totals per phase accumulate in the module global
g_acc (read back by tools/passrun).  Phases, per group g: 3g = wait/barrier
before the loads + loads issued, 3g+1 = gates, 3g+2 = stores (+ barriers).

    python tools/phase_patch.py pass.cu out.cu
"""
import re
import sys


def patch(src):
    lines = src.split("\n")
    out = []
    ph = 0
    names = []
    for i, ln in enumerate(lines):
        if ln.startswith("__constant__ double kc["):
            out.append("__device__ unsigned long long g_acc[64];")
            out.append("#define STAMP(k) do { long long t_ = clock64(); if ((threadIdx.x & 31) == 0) sacc[(k) * 8 + (threadIdx.x >> 5)] += t_ - last; last = t_; } while (0)")
        if ln.startswith("int it = 0;"):
            out.append("__shared__ long long sacc[64 * 8]; for (int q = threadIdx.x; q < 64 * 8; q += blockDim.x) sacc[q] = 0; __syncthreads(); long long last = clock64();")
        m = re.match(r"\{ // group (\d+)", ln)
        if m:
            g = int(m.group(1))
            out.append(ln)
            continue
        if ln.startswith("d2 ph = mk("):
            out.append(f"STAMP({ph});")
            names.append(f"g{g} wait+loads")
            ph += 1
        if ln.startswith("unsigned b0") or ln.startswith("unsigned s0 ="):
            # barrier line before it belongs to the store phase
            if out[-1].startswith("__syncthreads();") or out[-1].startswith("__syncwarp();"):
                bar = out.pop()
                out.append(f"STAMP({ph});")
                out.append(bar)
            else:
                out.append(f"STAMP({ph});")
            names.append(f"g{g} gates")
            ph += 1
        out.append(ln)
        if ln == "}" and i + 1 < len(lines) and (re.match(r"\{ // group", lines[i + 1]) or lines[i + 1] == "}"):
            if names and names[-1].endswith("gates"):
                out.insert(len(out) - 1, f"STAMP({ph});")
                names.append(f"g{g} stores")
                ph += 1
    # flush at the end of the kernel: before the final wait_group line
    k = max(i for i, ln in enumerate(out) if "cp.async.wait_group 0" in ln)
    out.insert(k, "__syncthreads(); if (threadIdx.x < 64) { long long s_ = 0; for (int w = 0; w < 8; ++w) s_ += sacc[threadIdx.x * 8 + w]; if (s_) atomicAdd(&g_acc[threadIdx.x], (unsigned long long)s_); }")
    sys.stderr.write("phases: " + ", ".join(f"{i}={n}" for i, n in enumerate(names)) + "\n")
    return "\n".join(out)


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))
