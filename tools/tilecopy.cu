// tilecopy.cu -- HBM efficiency of the fused-pass access pattern, no gates.
//
// A fused pass reads a 2^11-amplitude tile whose low `flow` bits are
// contiguous (rows of 2^flow x 16 B) and whose other bits are arbitrary
// qubits, then writes it back in place.  This measures how fast HBM serves
// that pattern as a function of the row width and of which qubits the row
// bits are, to separate the memory-system bound from the kernel's own.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tilecopy tools/tilecopy.cu
//   ./tilecopy            (n = 26, 2^26 complex128 = 1 GiB)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

struct Map {
    int flow;
    int rowbit[11];
    int ncomp;
    int comp[40];
};

__global__ void __launch_bounds__(128) k_tilecopy(double2 *__restrict__ a, long long ntiles, Map M, double scale) {
    const int tid = threadIdx.x;
    const int colmask = (1 << M.flow) - 1;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        long long base = 0;
        for (int j = 0; j < M.ncomp; ++j)
            if ((t >> j) & 1) base |= 1ll << M.comp[j];
        double2 v[16];
        long long off[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int e = tid + k * 128;
            long long o = base + (e & colmask);
            int r = e >> M.flow;
            for (int j = 0; j < 11 - M.flow; ++j)
                if ((r >> j) & 1) o |= 1ll << M.rowbit[j];
            off[k] = o;
            v[k] = __ldcs(a + o);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            v[k].x *= scale;
            v[k].y *= scale;
            __stcs(a + off[k], v[k]);
        }
    }
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 26;
    const long long N = 1ll << n;
    double2 *a;
    cudaMalloc(&a, N * sizeof(double2));
    cudaMemset(a, 0, N * sizeof(double2));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, int flow, std::vector<int> rows, int ctas) {
        Map M{};
        M.flow = flow;
        std::vector<int> used(n, 0);
        for (int b = 0; b < flow; ++b) used[b] = 1;
        for (int j = 0; j < 11 - flow; ++j) {
            M.rowbit[j] = rows[j];
            used[rows[j]] = 1;
        }
        M.ncomp = 0;
        for (int b = 0; b < n; ++b)
            if (!used[b]) M.comp[M.ncomp++] = b;
        long long ntiles = N >> 11;
        int grid = (int)std::min<long long>(ntiles, (long long)sms * ctas);
        for (int w = 0; w < 3; ++w) k_tilecopy<<<grid, 128>>>(a, ntiles, M, 1.0);
        cudaEventRecord(e0);
        const int reps = 10;
        for (int r = 0; r < reps; ++r) k_tilecopy<<<grid, 128>>>(a, ntiles, M, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double gbs = 2.0 * N * 16 * reps / (ms * 1e-3) / 1e9;
        printf("%-34s flow=%d ctas/SM=%d  %8.1f GB/s  (%.3f ms/pass)\n", name, flow, ctas, gbs, ms / reps);
    };
    for (int ctas : {4, 8}) {
        run("contiguous rows", 3, {3, 4, 5, 6, 7, 8, 9, 10}, ctas);
        run("high rows 18-25", 3, {18, 19, 20, 21, 22, 23, 24, 25}, ctas);
        run("mixed rows (bench pass)", 3, {6, 7, 8, 11, 14, 17, 19, 20}, ctas);
        run("high rows flow4", 4, {19, 20, 21, 22, 23, 24, 25}, ctas);
        run("mixed rows flow4", 4, {6, 7, 8, 11, 14, 17, 19}, ctas);
        run("high rows flow5", 5, {20, 21, 22, 23, 24, 25}, ctas);
        run("mixed rows flow5", 5, {6, 7, 8, 11, 14, 17}, ctas);
        run("flow2 mixed", 2, {6, 7, 8, 11, 14, 17, 19, 20, 21}, ctas);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error: %s\n", cudaGetErrorString(err));
    return 0;
}
