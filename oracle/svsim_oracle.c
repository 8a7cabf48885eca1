/*
 * svsim_oracle.c -- CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so, and only as the
 * checker or the timed CPU baseline.
 *
 * It restates, in plain C99, the arithmetic of the reference package `svsim`
 * (read-only at /root/reference/pkg):
 *
 *   pair update      a[b0]        = q11*lo + q12*hi
 *                    a[b0+2^t]    = q21*lo + q22*hi
 *                    (kernel/_stride_cy.pyx:16-21, kernel/__init__.py:78-80)
 *   collapsed sweep  base = ((q>>t)<<(t+1)) | (q & (2^t-1)), q in [0, N/2)
 *                    (kernel/_stride_cy.pyx:51-54)
 *   controlled       same sweep, pair skipped unless (base>>c)&1
 *                    (kernel/_stride_cy.pyx:86-90)
 *   own-row exchange low rank  a[j] = q11*mine + q12*other
 *                    high rank a[j] = q21*other + q22*mine
 *                    (engine.py:249-254, scheme b; engine.py:272 chunked)
 *   norm2            sum |a_j|^2 (core.py:171-174)
 *
 * Build flags mirror the reference's setup.py:43-50: -O3 -fopenmp
 * -ffp-contract=off, so every complex product is (ac-bd, ad+bc) with no
 * fused multiply-add and the results are bit-identical to the compiled
 * reference kernel (verified against oracle/_ref and tests/golden).
 */
#include <complex.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double _Complex dc;

static inline dc load_q(const double *q, int k) { return CMPLX(q[2 * k], q[2 * k + 1]); }

/* _stride_cy.pyx:16-21 */
static inline void pair(dc *a, int64_t b0, int64_t stride, dc q11, dc q12, dc q21, dc q22)
{
    dc lo = a[b0];
    dc hi = a[b0 + stride];
    a[b0] = q11 * lo + q12 * hi;
    a[b0 + stride] = q21 * lo + q22 * hi;
}

/* Single-qubit gate on target t, in place.  q = re/im of q11 q12 q21 q22.
 * workers <= 1: sequential block sweep (_stride_cy.pyx:33-38); otherwise the
 * collapsed prange sweep (_stride_cy.pyx:51-54).  Same pairs, same
 * arithmetic, so both are bit-identical. */
void or_apply_single(double *amps, int64_t n_amps, const double *q, int t, int workers)
{
    dc *a = (dc *)amps;
    dc q11 = load_q(q, 0), q12 = load_q(q, 1), q21 = load_q(q, 2), q22 = load_q(q, 3);
    int64_t stride = (int64_t)1 << t;
    int64_t npairs = n_amps >> 1;
    if (workers <= 1) {
        int64_t nblocks = n_amps >> (t + 1);
        for (int64_t b = 0; b < nblocks; ++b) {
            int64_t j = b << (t + 1);
            for (int64_t l = j; l < j + stride; ++l) pair(a, l, stride, q11, q12, q21, q22);
        }
        return;
    }
#pragma omp parallel for schedule(static) num_threads(workers)
    for (int64_t qq = 0; qq < npairs; ++qq) {
        int64_t base = ((qq >> t) << (t + 1)) | (qq & (stride - 1));
        pair(a, base, stride, q11, q12, q21, q22);
    }
}

/* `reps` consecutive applications of the same single-qubit gate on target t
 * (BASELINE configs[2]: 10 repetitions per target).  Each application
 * updates every pair (base, base+2^t) from that pair's own two amplitudes
 * only, so applying all `reps` to one pair before moving to the next pair is
 * bit-identical to `reps` full sweeps of or_apply_single -- it only keeps
 * the pair in registers (a checker speed-up; same arithmetic, same order per
 * amplitude). */
void or_apply_single_reps(double *amps, int64_t n_amps, const double *q, int t, int reps, int workers)
{
    dc *a = (dc *)amps;
    dc q11 = load_q(q, 0), q12 = load_q(q, 1), q21 = load_q(q, 2), q22 = load_q(q, 3);
    int64_t stride = (int64_t)1 << t;
    int64_t npairs = n_amps >> 1;
#pragma omp parallel for schedule(static) num_threads(workers > 0 ? workers : 1)
    for (int64_t qq = 0; qq < npairs; ++qq) {
        int64_t base = ((qq >> t) << (t + 1)) | (qq & (stride - 1));
        for (int r = 0; r < reps; ++r) pair(a, base, stride, q11, q12, q21, q22);
    }
}

/* Controlled gate: pair (base, base+2^t) updated only where bit c of base is
 * set (_stride_cy.pyx:57-90). */
void or_apply_controlled(double *amps, int64_t n_amps, const double *q, int c, int t, int workers)
{
    dc *a = (dc *)amps;
    dc q11 = load_q(q, 0), q12 = load_q(q, 1), q21 = load_q(q, 2), q22 = load_q(q, 3);
    int64_t stride = (int64_t)1 << t;
    int64_t npairs = n_amps >> 1;
    if (workers <= 1) {
        int64_t nblocks = n_amps >> (t + 1);
        for (int64_t b = 0; b < nblocks; ++b) {
            int64_t j = b << (t + 1);
            for (int64_t l = j; l < j + stride; ++l)
                if ((l >> c) & 1) pair(a, l, stride, q11, q12, q21, q22);
        }
        return;
    }
#pragma omp parallel for schedule(static) num_threads(workers)
    for (int64_t qq = 0; qq < npairs; ++qq) {
        int64_t base = ((qq >> t) << (t + 1)) | (qq & (stride - 1));
        if ((base >> c) & 1) pair(a, base, stride, q11, q12, q21, q22);
    }
}

/* Own-row exchange update of the paper's single-amplitude protocol
 * (engine.py:241-254) applied to a whole slab: `other` holds the partner
 * rank's amplitudes at the same local indices.  cbit < 0: every index;
 * otherwise only local indices with bit cbit set (engine.py:199-203, 244). */
void or_exchange_own_row(double *own, const double *other, int64_t count, const double *q,
                         int own_is_low, int cbit)
{
    dc *a = (dc *)own;
    const dc *o = (const dc *)other;
    dc q11 = load_q(q, 0), q12 = load_q(q, 1), q21 = load_q(q, 2), q22 = load_q(q, 3);
    for (int64_t j = 0; j < count; ++j) {
        if (cbit >= 0 && !((j >> cbit) & 1)) continue;
        dc mine = a[j];
        dc oth = o[j];
        a[j] = own_is_low ? (q11 * mine + q12 * oth) : (q21 * oth + q22 * mine);
    }
}

/* sum_j |a_j|^2 in index order (core.py:171-174 computes vdot(a,a).real;
 * summation order differs from numpy's pairwise sum by rounding only). */
double or_norm2(const double *amps, int64_t n_amps)
{
    double s = 0.0;
    for (int64_t j = 0; j < n_amps; ++j) {
        double re = amps[2 * j], im = amps[2 * j + 1];
        s += re * re + im * im;
    }
    return s;
}

/* probs[j] = |a_j|^2 = re*re + im*im (the measured-probability vector,
 * abs(gather(ds).amps)**2; SURVEY 8(a) note). */
void or_probs(const double *amps, int64_t n_amps, double *probs)
{
    for (int64_t j = 0; j < n_amps; ++j) {
        double re = amps[2 * j], im = amps[2 * j + 1];
        probs[j] = re * re + im * im;
    }
}

int or_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
