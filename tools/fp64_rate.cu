// fp64_rate.cu -- FP64 pipe microbenchmark: DFMA issue rate per SM sub-partition
// as a function of warps per scheduler and independent chains per thread.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/bin/fp64_rate tools/fp64_rate.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int ILP, int KIND>
__global__ void __launch_bounds__(128) k(double *out, double a, double b, int iters) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int i = 0; i < ILP; ++i) {
                if (KIND == 0) x[i] = __fma_rn(x[i], a, b);
                if (KIND == 1) x[i] = __dadd_rn(x[i], b);
                if (KIND == 2) x[i] = __dmul_rn(x[i], a);
                if (KIND == 3) x[i] = __fma_rn(x[i], x[(i + 1) % ILP], x[(i + 2) % ILP]);  // three register operands
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

template <int ILP, int KIND>
void run(const char *name, int sms, double clk_ghz) {
    double *out;
    cudaMalloc(&out, 8);
    const int iters = 2000;
    for (int cps = 1; cps <= 8; cps *= 2) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k<ILP, KIND><<<sms * cps, 128>>>(out, 1.0000001, 1e-9, iters);
        cudaEventRecord(e0);
        k<ILP, KIND><<<sms * cps, 128>>>(out, 1.0000001, 1e-9, iters);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double instr_per_sched = double(iters) * 8 * ILP * cps;  // warp-instructions per scheduler
        double cyc = ms * 1e-3 * clk_ghz * 1e9;
        printf("%-10s ILP %2d warps/sched %d: %.3f ms  %.2f cycles per warp-instr per scheduler (at %.2f GHz)  %.1f TFLOP/s-equiv\n",
               name, ILP, cps, ms, cyc / instr_per_sched, clk_ghz,
               (KIND == 0 || KIND == 3 ? 2.0 : 1.0) * instr_per_sched * 4 * sms * 32 / (ms * 1e-3) / 1e12);
    }
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int sms = p.multiProcessorCount;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    double ghz = khz * 1e-6;
    printf("%s, %d SMs, clock attr %.3f GHz\n", p.name, sms, ghz);
    run<4, 0>("dfma", sms, ghz);
    run<8, 0>("dfma", sms, ghz);
    run<16, 0>("dfma", sms, ghz);
    run<16, 1>("dadd", sms, ghz);
    run<16, 2>("dmul", sms, ghz);
    run<16, 3>("dfma3reg", sms, ghz);
    return 0;
}
