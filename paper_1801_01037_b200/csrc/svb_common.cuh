// svb_common.cuh -- shared device math, gate classification and index helpers.
//
// Complex arithmetic is written with explicit round-to-nearest intrinsics so
// nvcc can never contract a multiply-add: a product is (ac - bd, ad + bc),
// exactly what the reference's C99 `double _Complex` code computes under
// -ffp-contract=off (_stride_cy.pyx:16-21; setup.py:46-48).
//
// Gate kinds: a kernel may skip terms whose coefficient is exactly zero and
// multiply real / imaginary coefficients with two products instead of four.
// Each shortcut returns the same bits as the full formula (a product with a
// zero component contributes a signed zero, and x + (+-0) == x), except that
// a zero result may carry the other sign -- invisible to == and to max-abs
// error.  So every kind is bit-compatible with the reference.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace svb {

enum Kind : int {
    K_GENERAL = 0,  // all four entries complex
    K_REAL = 1,     // all entries real (H, X, Z, Ry, I)
    K_DIAG = 2,     // q12 = q21 = 0   (Z, S, T, Rz, phase)
    K_ANTI = 3,     // q11 = q22 = 0   (X, Y)
    K_RX = 4,       // q11, q22 real; q12, q21 imaginary (Rx)
};

struct Gate {
    double2 m[4];  // q11 q12 q21 q22
    int kind;
    int d0_one;    // q11 == 1 exactly (diag gates touch only the |1> half)
};

__host__ inline Gate make_gate(const double q[8]) {
    Gate g;
    for (int i = 0; i < 4; ++i) g.m[i] = make_double2(q[2 * i], q[2 * i + 1]);
    auto isz = [](double2 z) { return z.x == 0.0 && z.y == 0.0; };
    auto isr = [](double2 z) { return z.y == 0.0; };
    auto isi = [](double2 z) { return z.x == 0.0; };
    bool allreal = isr(g.m[0]) && isr(g.m[1]) && isr(g.m[2]) && isr(g.m[3]);
    if (isz(g.m[1]) && isz(g.m[2]))
        g.kind = K_DIAG;
    else if (isz(g.m[0]) && isz(g.m[3]))
        g.kind = K_ANTI;
    else if (allreal)
        g.kind = K_REAL;
    else if (isr(g.m[0]) && isr(g.m[3]) && isi(g.m[1]) && isi(g.m[2]))
        g.kind = K_RX;
    else
        g.kind = K_GENERAL;
    g.d0_one = (g.m[0].x == 1.0 && g.m[0].y == 0.0);
    return g;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
// (r + 0i) * x == (r*x.re, r*x.im)
__device__ __forceinline__ double2 rmul(double r, double2 x) {
    return make_double2(__dmul_rn(r, x.x), __dmul_rn(r, x.y));
}
// (0 + s i) * x == (-(s*x.im), s*x.re)
__device__ __forceinline__ double2 imul(double s, double2 x) {
    return make_double2(-__dmul_rn(s, x.y), __dmul_rn(s, x.x));
}

// Row update: out = ca*lo + cb*hi, with ca/cb the row's coefficients.
// `hi_row` selects the second row (q21, q22) instead of the first (q11, q12).
template <int KIND>
__device__ __forceinline__ double2 row(const Gate &g, bool hi_row, double2 lo, double2 hi) {
    const double2 ca = hi_row ? g.m[2] : g.m[0];
    const double2 cb = hi_row ? g.m[3] : g.m[1];
    if (KIND == K_GENERAL) return cadd(cmul(ca, lo), cmul(cb, hi));
    if (KIND == K_REAL) return cadd(rmul(ca.x, lo), rmul(cb.x, hi));
    if (KIND == K_DIAG) return hi_row ? cmul(cb, hi) : cmul(ca, lo);
    if (KIND == K_ANTI) return hi_row ? cmul(ca, lo) : cmul(cb, hi);
    // K_RX: first row real*lo + imag*hi, second row imag*lo + real*hi
    if (hi_row) return cadd(imul(ca.y, lo), rmul(cb.x, hi));
    return cadd(rmul(ca.x, lo), imul(cb.y, hi));
}

// Both rows with the coefficients passed by value (keeps them in registers).
template <int KIND>
__device__ __forceinline__ void pair_both_c(double2 q11, double2 q12, double2 q21, double2 q22,
                                            double2 &lo, double2 &hi) {
    const double2 a = lo, b = hi;
    if (KIND == K_GENERAL) {
        lo = cadd(cmul(q11, a), cmul(q12, b));
        hi = cadd(cmul(q21, a), cmul(q22, b));
    } else if (KIND == K_REAL) {
        lo = cadd(rmul(q11.x, a), rmul(q12.x, b));
        hi = cadd(rmul(q21.x, a), rmul(q22.x, b));
    } else if (KIND == K_DIAG) {
        lo = cmul(q11, a);
        hi = cmul(q22, b);
    } else if (KIND == K_ANTI) {
        lo = cmul(q12, b);
        hi = cmul(q21, a);
    } else {  // K_RX
        lo = cadd(rmul(q11.x, a), imul(q12.y, b));
        hi = cadd(imul(q21.y, a), rmul(q22.x, b));
    }
}

// FMA-contracted variants (SVB_RUN_FMA): fewer FP64 instructions and one
// rounding per output component instead of up to three; NOT bit-identical to
// the reference, agrees to ~1 ulp.
__device__ __forceinline__ double2 cmul_f(double2 a, double2 b) {
    return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

template <int KIND>
__device__ __forceinline__ void pair_both_fma(double2 q11, double2 q12, double2 q21, double2 q22,
                                              double2 &lo, double2 &hi) {
    const double2 a = lo, b = hi;
    if (KIND == K_GENERAL) {
        lo = make_double2(__fma_rn(q11.x, a.x, __fma_rn(-q11.y, a.y, __fma_rn(q12.x, b.x, -__dmul_rn(q12.y, b.y)))),
                          __fma_rn(q11.x, a.y, __fma_rn(q11.y, a.x, __fma_rn(q12.x, b.y, __dmul_rn(q12.y, b.x)))));
        hi = make_double2(__fma_rn(q21.x, a.x, __fma_rn(-q21.y, a.y, __fma_rn(q22.x, b.x, -__dmul_rn(q22.y, b.y)))),
                          __fma_rn(q21.x, a.y, __fma_rn(q21.y, a.x, __fma_rn(q22.x, b.y, __dmul_rn(q22.y, b.x)))));
    } else if (KIND == K_REAL) {
        lo = make_double2(__fma_rn(q11.x, a.x, __dmul_rn(q12.x, b.x)), __fma_rn(q11.x, a.y, __dmul_rn(q12.x, b.y)));
        hi = make_double2(__fma_rn(q21.x, a.x, __dmul_rn(q22.x, b.x)), __fma_rn(q21.x, a.y, __dmul_rn(q22.x, b.y)));
    } else if (KIND == K_DIAG) {
        lo = cmul_f(q11, a);
        hi = cmul_f(q22, b);
    } else if (KIND == K_ANTI) {
        lo = cmul_f(q12, b);
        hi = cmul_f(q21, a);
    } else {  // K_RX: q11, q22 real; q12, q21 imaginary
        lo = make_double2(__fma_rn(q11.x, a.x, -__dmul_rn(q12.y, b.y)), __fma_rn(q11.x, a.y, __dmul_rn(q12.y, b.x)));
        hi = make_double2(__fma_rn(q22.x, b.x, -__dmul_rn(q21.y, a.y)), __fma_rn(q22.x, b.y, __dmul_rn(q21.y, a.x)));
    }
}

template <int KIND>
__device__ __forceinline__ void pair_both(const Gate &g, double2 &lo, double2 &hi) {
    double2 a = lo, b = hi;
    lo = row<KIND>(g, false, a, b);
    hi = row<KIND>(g, true, a, b);
}

// Insert a bit of value v at position pos of x (bits >= pos move up by one).
__device__ __host__ __forceinline__ int64_t insert_bit(int64_t x, int pos, int v) {
    int64_t low = x & ((int64_t(1) << pos) - 1);
    return ((x >> pos) << (pos + 1)) | (int64_t(v) << pos) | low;
}

__device__ __forceinline__ double2 shfl_xor_d2(double2 v, int m) {
    v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
    v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
    return v;
}

}  // namespace svb

// error plumbing and launch accounting shared by the host side
namespace svb {
enum ProfClass : int {
    PROF_PAIR_HIGH = 0,  // k_pair_high: target >= 5
    PROF_PAIR_LOW = 1,   // k_pair_low: target < 5, SHFL own-row
    PROF_DIAG = 2,       // k_diag: elementwise diagonal gates
    PROF_TINY = 3,       // k_tiny: < 64 amplitudes
    PROF_FUSED = 4,      // k_fused: multi-gate shared-memory pass
    PROF_EXCHANGE = 5,   // k_exchange_own_row / k_pair_update
    PROF_NORM = 6,       // norm / probs
    PROF_FUSED_JIT = 7,  // kpass: NVRTC-specialised fused pass (jit.cu)
    PROF_DENSE = 8,      // k_dense_embed / k_dense_matvec (dense verifier)
    PROF_SYNC = 9,       // k_signal: pairwise rank sync of the peer transport
    PROF_SWAPNET = 10,   // k_swap_bits: a trailing SWAP network in one pass (fused.cu)
    PROF_NCLASSES = 11
};
struct LaunchInfo {
    int kernels;
    int cls;
    int64_t alg_bytes;
};
// profiler: when enabled, launches made through these hooks are bracketed
// by CUDA events on their stream and aggregated per class
bool prof_on();
void prof_begin(cudaStream_t s);
void prof_end(cudaStream_t s, const LaunchInfo &li);
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *where);
}  // namespace svb

#define SVB_CHECK_LAUNCH(where)                                        \
    do {                                                               \
        cudaError_t _e = cudaGetLastError();                           \
        if (_e != cudaSuccess) return ::svb::cuda_status(_e, where);   \
    } while (0)
