// fp64_lds_overlap.cu -- do FP64 arithmetic and shared-memory traffic overlap on
// one SM?  Streams of independent DFMAs and of conflict-free LDS.128 /
// STS.128, alone, interleaved in every warp, and split over warps (half the
// warps do arithmetic, half shared memory), at 8 warps per SM like a pass.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/bin/fp64_lds_overlap tools/fp64_lds_overlap.cu
#include <cuda_runtime.h>
#include <cstdio>

// mode bit 0: this warp does FP64; bit 1: this warp does shared memory
template <int NF, int NL>
__global__ void __launch_bounds__(256) k(double *out, double a, double b, int iters, int split) {
    extern __shared__ double2 sm[];
    const int warp = threadIdx.x >> 5;
    bool do_f = NF > 0, do_l = NL > 0;
    if (split && NF > 0 && NL > 0) {
        do_f = (warp & 1) == 0;   // even warps: arithmetic; odd warps: shared memory
        do_l = !do_f;
    }
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    double2 acc = make_double2(0, 0);
    double2 *p = sm + threadIdx.x;  // 16 B per lane, consecutive lanes: conflict-free
    for (int it = 0; it < iters; ++it) {
        if (do_f && do_l) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
#pragma unroll
                for (int i = 0; i < NF / 8; ++i) x[i % 16] = __fma_rn(x[i % 16], a, b);
#pragma unroll
                for (int i = 0; i < NL / 8; ++i) {
                    double2 v = p[((r * (NL / 8) + i) & 15) * 256];
                    acc.x += v.x == 12345.0 ? 1.0 : 0.0;  // cheap consumer, rarely true
                }
            }
        } else if (do_f) {
#pragma unroll
            for (int i = 0; i < NF; ++i) x[i % 16] = __fma_rn(x[i % 16], a, b);
        } else if (do_l) {
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                double2 v = p[(i & 15) * 256];
                acc.x += v.x == 12345.0 ? 1.0 : 0.0;
            }
        }
    }
    double s = acc.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

template <int NF, int NL>
float run(int sms, int iters, int split) {
    double *out;
    cudaMalloc(&out, 8);
    cudaFuncSetAttribute(k<NF, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<NF, NL><<<sms, 256, 65536>>>(out, 1.0000001, 1e-9, iters, split);
    cudaEventRecord(e0);
    k<NF, NL><<<sms, 256, 65536>>>(out, 1.0000001, 1e-9, iters, split);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    return ms;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount, iters = 4000;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double cyc = khz * 1e3 * 1e-3 / iters;  // cycles per iteration per ms
    // per iteration and warp: 256 DFMA (2 cycles each on the scheduler's pipe: 512 cycles,
    // 2 warps per scheduler: 1024) and 64 LDS.128 (512 B each; 8 warps: 256 KB per iteration
    // per SM = 2048 cycles at 128 B/clk)
    float f = run<256, 0>(sms, iters, 0), l = run<0, 64>(sms, iters, 0);
    float both = run<256, 64>(sms, iters, 0), split = run<256, 64>(sms, iters, 1);
    printf("8 warps/SM, per iteration: 256 DFMA and / or 64 LDS.128 per warp\n");
    printf("FP64 only            %.3f ms  %.0f cycles per iteration\n", f, f * cyc);
    printf("LDS only             %.3f ms  %.0f cycles per iteration\n", l, l * cyc);
    printf("both, every warp     %.3f ms  %.0f cycles per iteration (sum of the two alone: %.0f, max: %.0f)\n", both, both * cyc,
           (f + l) * cyc, (f > l ? f : l) * cyc);
    printf("split over warps     %.3f ms  %.0f cycles per iteration (even warps FP64, odd warps LDS: half the work of each kind)\n",
           split, split * cyc);
    float f2 = run<128, 0>(sms, iters, 0), l2 = run<0, 32>(sms, iters, 0), both2 = run<128, 32>(sms, iters, 0);
    printf("half sizes: FP64 %.0f  LDS %.0f  both %.0f cycles per iteration\n", f2 * cyc, l2 * cyc, both2 * cyc);
    return 0;
}
