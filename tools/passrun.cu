// passrun.cu -- time ONE specialised pass (a cubin SVB_JIT_DUMP wrote, or a
// hand-edited variant of its source compiled with nvcc -cubin) on a 2^n
// state, outside the library: the experiment loop for kernel-structure
// questions (CTAs per SM, grid size, barriers, prefetch variants).
//
//   nvcc -O2 -o tools/bin/passrun tools/passrun.cu -lcuda
//   passrun pass76.cubin n fm threads smem_bytes ctas_per_sm reps [label]
//
// Prints: label, grid, average ms per launch, GB/s of algorithmic bytes
// (32 B per amplitude).  The state (16 B x 2^n) is far larger than L2 at the
// sizes used (n = 26: 1 GiB).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        CUresult r_ = (x);                                                             \
        if (r_ != CUDA_SUCCESS) {                                                      \
            const char *s_ = nullptr;                                                  \
            cuGetErrorString(r_, &s_);                                                 \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?"); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

int main(int argc, char **argv) {
    if (argc < 8) {
        fprintf(stderr, "usage: passrun cubin n fm threads smem ctas_per_sm reps [label]\n");
        return 2;
    }
    const char *path = argv[1];
    const int n = atoi(argv[2]), fm = atoi(argv[3]), threads = atoi(argv[4]), smem = atoi(argv[5]);
    const double cps = atof(argv[6]);
    const int reps = atoi(argv[7]);
    const char *label = argc > 8 ? argv[8] : path;
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    if (const char *g = getenv("PASSRUN_L2_FETCH")) {  // experiment: L2 fetch granularity (32 / 64 / 128 B)
        CK(cuCtxSetLimit(CU_LIMIT_MAX_L2_FETCH_GRANULARITY, (size_t)atoi(g)));
        size_t v = 0;
        cuCtxGetLimit(&v, CU_LIMIT_MAX_L2_FETCH_GRANULARITY);
        fprintf(stderr, "L2 fetch granularity %zu\n", v);
    }
    int sms = 0;
    CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
    CUmodule mod;
    CK(cuModuleLoad(&mod, path));
    CUfunction fn;
    CK(cuModuleGetFunction(&fn, mod, "kpass"));
    if (smem > 0) CK(cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem));
    const size_t N = size_t(1) << n;
    CUdeviceptr a;
    CK(cuMemAlloc(&a, N * 16));
    {
        // a bounded non-trivial pattern (values do not change FP64 timing)
        std::vector<double> h(1 << 20);
        for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-4 * double((i * 2654435761u) % 1000) - 0.05;
        for (size_t off = 0; off < N * 16; off += h.size() * 8) CK(cuMemcpyHtoD(a + off, h.data(), h.size() * 8));
    }
    long long ntiles = (long long)(N >> fm);
    int grid = (int)(cps * sms + 0.5);
    if (grid > ntiles) grid = (int)ntiles;
    void *args[] = {&a, &ntiles};
    CUdeviceptr ctr = 0;  // dynamic tile scheduling variants (tools/dyn_patch.py): zeroed before every launch
    {
        size_t cb = 0;
        if (cuModuleGetGlobal(&ctr, &cb, mod, "g_ctr") != CUDA_SUCCESS) ctr = 0;
    }
    CUevent e0, e1;
    CK(cuEventCreate(&e0, 0));
    CK(cuEventCreate(&e1, 0));
    for (int i = 0; i < 3; ++i) {
        if (ctr) CK(cuMemsetD32Async(ctr, 0, 1, 0));
        CK(cuLaunchKernel(fn, grid, 1, 1, threads, 1, 1, smem, 0, args, nullptr));
    }
    CK(cuCtxSynchronize());
    CK(cuEventRecord(e0, 0));
    for (int i = 0; i < reps; ++i) {
        if (ctr) CK(cuMemsetD32Async(ctr, 0, 1, 0));
        CK(cuLaunchKernel(fn, grid, 1, 1, threads, 1, 1, smem, 0, args, nullptr));
    }
    CK(cuEventRecord(e1, 0));
    CK(cuCtxSynchronize());
    float ms = 0;
    CK(cuEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("%-44s grid %4d  %8.4f ms  %7.1f GB/s\n", label, grid, ms, 32.0 * double(N) / (ms * 1e6));
    {
        // phase stamps of an instrumented variant (tools/phase_patch.py): cycles per warp per tile
        CUdeviceptr g;
        size_t gb = 0;
        if (cuModuleGetGlobal(&g, &gb, mod, "g_acc") == CUDA_SUCCESS && gb >= 64 * 8) {
            unsigned long long acc[64];
            CK(cuMemcpyDtoH(acc, g, sizeof acc));
            const double per = double(reps + 3) * double(ntiles) * (threads / 32);
            double tot = 0;
            for (int q = 0; q < 64; ++q) tot += double(acc[q]);
            printf("  cycles per warp per tile, by phase (total %.0f):", tot / per);
            for (int q = 0; q < 64; ++q)
                if (acc[q]) printf(" %d:%.0f", q, double(acc[q]) / per);
            printf("\n");
        }
    }
    {
        // per-CTA timeline of an instrumented variant (tools/trace_patch.py), last launch
        CUdeviceptr g;
        size_t gb = 0;
        if (cuModuleGetGlobal(&g, &gb, mod, "g_trace") == CUDA_SUCCESS) {
            std::vector<long long> tr(gb / 8);
            CK(cuMemcpyDtoH(tr.data(), g, gb));
            for (int sm = 0; sm < 4; ++sm) {
                const long long t0 = std::min(tr[((sm * 2 + 0) * 2 + 0) * 64], tr[((sm * 2 + 1) * 2 + 0) * 64]);
                for (int slot = 0; slot < 2; ++slot) {
                    printf("  SM %d CTA %d tile starts (cycles):", sm, slot);
                    for (int it = 0; it < 24; ++it) printf(" %lld", tr[((sm * 2 + slot) * 2 + 0) * 64 + it] - t0);
                    printf("\n  SM %d CTA %d last-group starts:    ", sm, slot);
                    for (int it = 0; it < 24; ++it) printf(" %lld", tr[((sm * 2 + slot) * 2 + 1) * 64 + it] - t0);
                    printf("\n");
                }
            }
        }
    }
    return 0;
}
