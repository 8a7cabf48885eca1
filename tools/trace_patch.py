"""Experiment: per-CTA timeline of a mode-2 pass.  Thread 0 of every CTA on
SMs 0..3 writes (smid, clock64) at the start of every tile and at the start of
its last group into the module global g_trace; tools/passrun prints, per SM,
the two resident CTAs' tile-start times so their relative phase is visible.

    python tools/trace_patch.py pass.cu out.cu
"""
import re
import sys


def patch(src):
    lines = src.split("\n")
    out = []
    gstarts = [i for i, ln in enumerate(lines) if re.match(r"\{ // group \d+", ln)]
    last = gstarts[-1]
    for i, ln in enumerate(lines):
        if ln.startswith("__constant__ double kc["):
            out.append("__device__ long long g_trace[4 * 2 * 2 * 64];  // [sm][cta slot][event][tile]")
            out.append("__device__ unsigned g_slot[4];")
        if ln.startswith("int it = 0;"):
            out.append("unsigned smid; asm volatile(\"mov.u32 %0, %%smid;\" : \"=r\"(smid));")
            out.append("__shared__ int tslot; if (threadIdx.x == 0) tslot = smid < 4 ? (int)atomicAdd(&g_slot[smid], 1u) & 1 : -1; __syncthreads();")
        out.append(ln)
        if ln.startswith("d2 *const pa = a + tbase(tix);"):
            out.append("if (threadIdx.x == 0 && tslot >= 0 && it < 64) g_trace[((smid * 2 + tslot) * 2 + 0) * 64 + it] = clock64();")
        if i == last:
            out.append("if (threadIdx.x == 0 && tslot >= 0 && it < 64) g_trace[((smid * 2 + tslot) * 2 + 1) * 64 + it] = clock64();")
    return "\n".join(out)


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))
