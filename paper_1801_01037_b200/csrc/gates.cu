// gates.cu -- one-HBM-pass kernels for a single (optionally controlled) 2x2 gate.
//
// Replaces the reference's stride sweep (_stride_cy.pyx:24-90): the same
// disjoint pairs (j, j + 2^t), bit t of j clear, same arithmetic, but laid out
// for HBM3e:
//
//  * "rows": 32 consecutive amplitudes = 512 B, one warp, one double2 (16 B)
//    per lane -> every load/store instruction moves four full 128 B lines.
//  * t >= 5 (k_pair_high): a work unit is the row pair (r, r + 2^(t-5));
//    each lane owns one amplitude pair and writes both rows.
//  * t < 5 (k_pair_low): the partner is inside the same row, lane ^ 2^t;
//    lanes swap values with SHFL and each computes ITS OWN row -- the
//    paper's own-row rule (engine.py:254) -- so loads stay fully coalesced.
//  * diagonal gates (Z S T Rz, controlled phase): k_diag is elementwise; with
//    q11 == 1 it visits only the |1> half (L/2 amplitudes, or L/4 under a
//    control), the algorithmic minimum.
//  * control bit c: c >= 5 selects rows (skipped rows are never read); c < 5
//    predicates lanes (skipped lanes neither load nor store).
//
// Each warp processes UPW units with all loads issued before any math
// (memory-level parallelism ~UPW x 2 x 16 B per lane in flight).
#include <cstdio>

#include "svb_common.cuh"

namespace svb {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;

// row index for work unit u: insert the target row bit (value 0) and, when
// the control is a row bit, the control row bit (value 1), low position first
__device__ __forceinline__ int64_t unit_row(int64_t u, int tb, int cb) {
    if (cb < 0) return tb < 0 ? u : insert_bit(u, tb, 0);
    if (tb < 0) return insert_bit(u, cb, 1);
    if (cb < tb) return insert_bit(insert_bit(u, cb, 1), tb, 0);
    return insert_bit(insert_bit(u, tb, 0), cb, 1);
}

template <int KIND, int UPW>
__global__ void __launch_bounds__(kThreads) k_pair_high(double2 *__restrict__ a, int64_t units,
                                                        Gate g, int t, int c) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int tb = t - 5;
    const int cb = c >= 5 ? c - 5 : -1;
    const bool lane_on = (c < 0 || c >= 5) ? true : ((lane >> c) & 1);
    const int64_t stride = int64_t(1) << t;
    double2 lo[UPW], hi[UPW];
    int64_t idx[UPW];
    bool on[UPW];
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
        int64_t u = warp * UPW + k;
        on[k] = lane_on && u < units;
        idx[k] = unit_row(u, tb, cb) * 32 + lane;
        if (on[k]) {
            lo[k] = a[idx[k]];
            hi[k] = a[idx[k] + stride];
        }
    }
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
        if (on[k]) {
            pair_both<KIND>(g, lo[k], hi[k]);
            a[idx[k]] = lo[k];
            a[idx[k] + stride] = hi[k];
        }
    }
}

template <int KIND, int UPW>
__global__ void __launch_bounds__(kThreads) k_pair_low(double2 *__restrict__ a, int64_t units,
                                                       Gate g, int t, int c) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int cb = c >= 5 ? c - 5 : -1;
    const bool lane_on = (c < 0 || c >= 5) ? true : ((lane >> c) & 1);
    const bool hi_row = (lane >> t) & 1;
    const int m = 1 << t;
    double2 v[UPW];
    int64_t idx[UPW];
    bool on[UPW];
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
        int64_t u = warp * UPW + k;
        bool valid = u < units;  // warp-uniform
        on[k] = lane_on && valid;
        idx[k] = unit_row(u, -1, cb) * 32 + lane;
        v[k] = on[k] ? a[idx[k]] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
        double2 other = shfl_xor_d2(v[k], m);
        double2 lo = hi_row ? other : v[k];
        double2 hi = hi_row ? v[k] : other;
        double2 r = row<KIND>(g, hi_row, lo, hi);
        if (on[k]) a[idx[k]] = r;
    }
}

// Elementwise diagonal gate: amplitude *= (bit t ? q22 : q11) on the indices
// whose `ones` bits are all set.  `ones` is sorted ascending, nones <= 3.
template <int UPT>
__global__ void __launch_bounds__(kThreads) k_diag(double2 *__restrict__ a, int64_t count, double2 d0,
                                                   double2 d1, int t, int nones, int o0, int o1,
                                                   int o2) {
    const int64_t base = (int64_t(blockIdx.x) * kThreads * UPT) + threadIdx.x;
    double2 v[UPT];
    int64_t idx[UPT];
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        int64_t e = base + int64_t(k) * kThreads;
        int64_t i = e;
        if (nones > 0) i = insert_bit(i, o0, 1);
        if (nones > 1) i = insert_bit(i, o1, 1);
        if (nones > 2) i = insert_bit(i, o2, 1);
        idx[k] = e < count ? i : -1;
        if (idx[k] >= 0) v[k] = a[i];
    }
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        if (idx[k] >= 0) {
            bool b = (idx[k] >> t) & 1;
            a[idx[k]] = cmul(b ? d1 : d0, v[k]);
        }
    }
}

// Tiny states (fewer than 64 amplitudes): one thread per pair.
__global__ void k_tiny(double2 *a, int64_t n_amps, Gate g, int t, int c) {
    int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= (n_amps >> 1)) return;
    int64_t b0 = insert_bit(q, t, 0);
    if (c >= 0 && !((b0 >> c) & 1)) return;
    double2 lo = a[b0], hi = a[b0 + (int64_t(1) << t)];
    pair_both<K_GENERAL>(g, lo, hi);
    a[b0] = lo;
    a[b0 + (int64_t(1) << t)] = hi;
}

template <int KIND>
static void launch_rows(double2 *a, int64_t n_amps, const Gate &g, int t, int c, cudaStream_t s) {
    constexpr int UPW_HIGH = 4;
    constexpr int UPW_LOW = 4;
    int64_t rows = n_amps >> 5;
    if (t >= 5) {
        int64_t units = rows >> 1;
        if (c >= 5) units >>= 1;
        int64_t warps = (units + UPW_HIGH - 1) / UPW_HIGH;
        int64_t blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
        k_pair_high<KIND, UPW_HIGH><<<(unsigned)blocks, kThreads, 0, s>>>(a, units, g, t, c);
    } else {
        int64_t units = rows;
        if (c >= 5) units >>= 1;
        int64_t warps = (units + UPW_LOW - 1) / UPW_LOW;
        int64_t blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
        k_pair_low<KIND, UPW_LOW><<<(unsigned)blocks, kThreads, 0, s>>>(a, units, g, t, c);
    }
}

// Launch one gate.  c < 0: single-qubit gate.  Returns the kernel class and
// the algorithmic HBM bytes of the launch (each touched amplitude read once
// and written once, 16 B each way).
LaunchInfo launch_gate(double2 *a, int64_t n_amps, const Gate &g, int t, int c, cudaStream_t s) {
    if (g.kind == K_DIAG && n_amps >= 64) {
        int ones[3], no = 0;
        if (c >= 0) ones[no++] = c;
        if (g.d0_one) ones[no++] = t;
        if (no == 2 && ones[0] > ones[1]) {
            int tmp = ones[0];
            ones[0] = ones[1];
            ones[1] = tmp;
        }
        int64_t count = n_amps >> no;
        constexpr int UPT = 4;
        int64_t blocks = (count + int64_t(kThreads) * UPT - 1) / (int64_t(kThreads) * UPT);
        k_diag<UPT><<<(unsigned)blocks, kThreads, 0, s>>>(a, count, g.m[0], g.m[3], t, no,
                                                          no > 0 ? ones[0] : 0,
                                                          no > 1 ? ones[1] : 0, 0);
        return LaunchInfo{1, PROF_DIAG, count * 32};
    }
    if (n_amps < 64) {
        k_tiny<<<1, 64, 0, s>>>(a, n_amps, g, t, c);
        return LaunchInfo{1, PROF_TINY, (c >= 0 ? n_amps / 2 : n_amps) * 32};
    }
    switch (g.kind) {
        case K_REAL: launch_rows<K_REAL>(a, n_amps, g, t, c, s); break;
        case K_DIAG: launch_rows<K_DIAG>(a, n_amps, g, t, c, s); break;
        case K_ANTI: launch_rows<K_ANTI>(a, n_amps, g, t, c, s); break;
        case K_RX: launch_rows<K_RX>(a, n_amps, g, t, c, s); break;
        default: launch_rows<K_GENERAL>(a, n_amps, g, t, c, s); break;
    }
    return LaunchInfo{1, t >= 5 ? PROF_PAIR_HIGH : PROF_PAIR_LOW, (c >= 0 ? n_amps / 2 : n_amps) * 32};
}

}  // namespace svb
