"""Experiment: dynamic tile scheduling for a mode-2 pass source.  A CTA takes
its first tile statically (blockIdx.x) and every further tile from a global
counter (thread 0 fetches the index of the tile after next right after the
tile-start barrier; everybody reads it behind the last group's barrier, where
the prefetch is issued), so the two CTAs of an SM -- the hardware scheduler
lets one of them run ~2x faster -- stop working only when the pass is out
of tiles.  tools/passrun zeroes g_ctr before every launch.

    python tools/dyn_patch.py pass.cu out.cu
"""
import sys


def patch(src):
    out = []
    for ln in src.split("\n"):
        if ln.startswith("__constant__ double kc["):
            out.append("__device__ unsigned g_ctr;")
        if ln.startswith("for (i64 tix = blockIdx.x; tix < ntiles; tix += gridDim.x, ++it) {"):
            out.append("__shared__ i64 s_next;")
            out.append("i64 nx = 0; unsigned tk = 0;")
            out.append("for (i64 tix = blockIdx.x; tix < ntiles; tix = nx, ++it) {")
            continue
        if ln.startswith("{ const i64 nx = tix + gridDim.x; if (nx < ntiles) fill("):
            # (the line before this one is the last group's barrier)
            bar = out.pop()
            out.append("if (threadIdx.x == 0) s_next = (i64)gridDim.x + tk;")
            out.append(bar)
            out.append("nx = s_next;")
            out.append("if (nx < ntiles) fill(reinterpret_cast<unsigned char *>(dsm), a + tbase(nx));")
            continue
        out.append(ln)
        if ln.startswith("__syncthreads();") and out[-2].startswith('asm volatile("cp.async.wait_group 0;'):
            out.append("if (threadIdx.x == 0) tk = atomicAdd(&g_ctr, 1u);")
    return "\n".join(out)


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))
