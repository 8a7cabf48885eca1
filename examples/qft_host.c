/* qft_host.c -- a compiled (non-Python) caller of libsvb.so through the C ABI
 * in include/svb.h only: builds the LSB-convention QFT on n qubits (H, then
 * controlled phases pi/2^(k-j), then the qubit-reversal swaps as three CNOTs
 * each -- the reference's form, workloads.qft_circuit), runs it on the host
 * array of a basis state |x> with svb_host_run_ops (H2D, fused passes, D2H)
 * and checks every amplitude against the closed form
 *     <y|QFT|x> = exp(2 pi i br(x) br(y) / 2^n) / 2^(n/2)
 * (SURVEY 8(c)), elementwise.  Exit status 0 iff max |error| <= 1e-12.
 *
 *   cc -O2 -Iinclude examples/qft_host.c -Lpaper_1801_01037_b200 -lsvb -lm -o qft_host
 *   LD_LIBRARY_PATH=paper_1801_01037_b200 ./qft_host [n] [x]
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "svb.h"

static void gate(svb_op *o, int kind, int t, int c, double q11r, double q11i, double q12r, double q12i,
                 double q21r, double q21i, double q22r, double q22i) {
    o->kind = kind;
    o->target = t;
    o->control = kind ? c : -1;
    o->reserved = 0;
    double q[8] = {q11r, q11i, q12r, q12i, q21r, q21i, q22r, q22i};
    for (int i = 0; i < 8; ++i) o->q[i] = q[i];
}

static uint64_t bitrev(uint64_t v, int n) {
    uint64_t r = 0;
    for (int i = 0; i < n; ++i) r |= ((v >> i) & 1) << (n - 1 - i);
    return r;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 16;
    const uint64_t N = (uint64_t)1 << n;
    const uint64_t x = argc > 2 ? strtoull(argv[2], 0, 0) % N : 0x2345 % N;
    const int nops = n + n * (n - 1) / 2 + 3 * (n / 2);
    svb_op *ops = calloc((size_t)nops, sizeof(svb_op));
    const double h = 1.0 / sqrt(2.0), pi = acos(-1.0);
    int k = 0;
    for (int j = 0; j < n; ++j) {
        gate(&ops[k++], 0, j, -1, h, 0, h, 0, h, 0, -h, 0);
        for (int t = j + 1; t < n; ++t) {
            const double phi = pi / (double)((uint64_t)1 << (t - j));
            gate(&ops[k++], 1, t, j, 1, 0, 0, 0, 0, 0, cos(phi), sin(phi));
        }
    }
    for (int p = 0; p < n / 2; ++p) {
        const int a = p, b = n - 1 - p;
        gate(&ops[k++], 1, b, a, 0, 0, 1, 0, 1, 0, 0, 0);
        gate(&ops[k++], 1, a, b, 0, 0, 1, 0, 1, 0, 0, 0);
        gate(&ops[k++], 1, b, a, 0, 0, 1, 0, 1, 0, 0, 0);
    }
    double *amps = calloc(2 * N, sizeof(double));
    amps[2 * x] = 1.0;
    int rc = svb_host_run_ops(amps, amps, (int64_t)N, ops, nops, SVB_RUN_FUSE | SVB_RUN_FMA | SVB_RUN_JIT);
    if (rc != SVB_OK) {
        fprintf(stderr, "svb_host_run_ops: %d %s\n", rc, svb_last_error());
        return 2;
    }
    double err = 0.0;
    const uint64_t bx = bitrev(x, n);
    for (uint64_t y = 0; y < N; ++y) {
        const uint64_t ph = (bx * bitrev(y, n)) & (N - 1);  /* exact in 64 bits for n <= 32 */
        const double ang = 2.0 * pi * (double)ph / (double)N, s = 1.0 / sqrt((double)N);
        const double dr = amps[2 * y] - s * cos(ang), di = amps[2 * y + 1] - s * sin(ang);
        const double e = sqrt(dr * dr + di * di);
        if (e > err) err = e;
    }
    printf("qft_host: n=%d x=%llu ops=%d max|err|=%.3e\n", n, (unsigned long long)x, nops, err);
    free(ops);
    free(amps);
    return err <= 1e-12 ? 0 : 1;
}
