// dense.cu -- the reference's dense-matrix verifier on the GPU (SURVEY
// §8(f)4; oracle.py:81-176): explicit 2^n x 2^n gate embeddings and
// row-by-row matrix-vector products, for n <= 12 (256 MiB of complex128).
//
// k_dense_embed writes one embedding: the identity except, for every row r
// with bit t clear (and bit c set when controlled), the 2x2 block
// [[q11 q12] [q21 q22]] at rows/columns (r, r | 2^t) -- the same entries
// embed_single's kron(I, kron(g, I)) and embed_controlled's index writes
// produce (oracle.py:81-116), bit for bit (every entry is 0, 1 or a gate
// entry).  One thread per 16 B entry, coalesced along the row.
//
// k_dense_matvec computes y = U x one warp per row: lane l accumulates
// columns l, l + 32, ... in ascending order with exact complex products
// (no FMA contraction, like the reference's C99 arithmetic), then a fixed
// xor-shuffle tree combines the lanes.  Each row's result depends only on
// that row, so any row partition (matvec_partitioned, oracle.py:154-176)
// reproduces matvec's bits exactly, as the reference's does.  HBM-bound:
// 16 B per matrix entry, read once.
#include "svb_common.cuh"

namespace svb {

__global__ void k_dense_embed(double2 *__restrict__ u, int64_t dim, Gate g, int t, int c) {
    const int64_t total = dim * dim;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / dim, col = e - r * dim;
        double2 v = make_double2(r == col ? 1.0 : 0.0, 0.0);
        const int64_t tb = int64_t(1) << t;
        const bool active = c < 0 || ((r >> c) & 1);
        // r and col in the same pair (differ at most in bit t), control set
        if (active && ((r ^ col) & ~tb) == 0) {
            const int rb = (r >> t) & 1, cb = (col >> t) & 1;
            v = g.m[rb * 2 + cb];
        }
        u[e] = v;
    }
}

__global__ void k_dense_matvec(const double2 *__restrict__ u, const double2 *__restrict__ x,
                               double2 *__restrict__ y, int64_t dim, int64_t row0, int64_t nrows) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t w = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nrows; w += warps) {
        const double2 *row = u + (row0 + w) * dim;
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t col = lane; col < dim; col += 32) {
            const double2 a = row[col], b = x[col];
            // (a.x b.x - a.y b.y, a.x b.y + a.y b.x), exact products
            acc = cadd(acc, make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                                         __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double2 p = make_double2(__shfl_xor_sync(0xffffffffu, acc.x, o),
                                           __shfl_xor_sync(0xffffffffu, acc.y, o));
            // lanes l and l ^ o add in a fixed order (lower lane first), so
            // both hold the same bits
            acc = (lane & o) ? cadd(p, acc) : cadd(acc, p);
        }
        if (lane == 0) y[row0 + w] = acc;
    }
}

LaunchInfo launch_dense_embed(double2 *u, int64_t dim, const Gate &g, int t, int c, cudaStream_t s) {
    const int64_t total = dim * dim;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
    k_dense_embed<<<(int)blocks, threads, 0, s>>>(u, dim, g, t, c);
    return LaunchInfo{1, PROF_DENSE, total * 16};
}

LaunchInfo launch_dense_matvec(const double2 *u, const double2 *x, double2 *y, int64_t dim, int64_t row0,
                               int64_t nrows, cudaStream_t s) {
    const int threads = 256;  // 8 rows per block
    const int64_t blocks = std::min<int64_t>((nrows + 7) / 8, 148 * 16);
    k_dense_matvec<<<(int)std::max<int64_t>(blocks, 1), threads, 0, s>>>(u, x, y, dim, row0, nrows);
    return LaunchInfo{1, PROF_DENSE, nrows * dim * 16 + dim * 16 + nrows * 16};
}

}  // namespace svb
