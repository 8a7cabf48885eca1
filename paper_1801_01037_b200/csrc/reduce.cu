// reduce.cu -- norm and probability kernels.
//
// norm2 (core.py:171-174, engine.py:453-454): two deterministic passes.
// Pass 1 runs a fixed grid of 148 x 8 blocks (one wave at 8 blocks/SM on
// B200's 148 SMs); each thread strides over the slab with 16 B double2
// loads, accumulates re^2 + im^2 in fp64, then warp shuffles and a
// shared-memory step reduce to one partial per block.  Pass 2 sums the
// partials in a fixed order in a single block, so the result is
// bit-reproducible run to run.
//
// probs: elementwise |a_j|^2 = re*re + im*im (the measured-probability
// vector, abs(gather(ds).amps)**2 in the reference's terms).
#include "svb_common.cuh"

namespace svb {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ double block_sum(double v) {
    __shared__ double part[kRedThreads / 32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < kRedThreads / 32 ? part[threadIdx.x] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

__global__ void __launch_bounds__(kRedThreads) k_norm_partial(const double2 *__restrict__ a,
                                                              int64_t n, double *partial) {
    double acc0 = 0.0, acc1 = 0.0;
    const int64_t stride = int64_t(gridDim.x) * kRedThreads;
    int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
    for (; i + stride < n; i += 2 * stride) {
        double2 x = a[i], y = a[i + stride];
        acc0 += x.x * x.x + x.y * x.y;
        acc1 += y.x * y.x + y.y * y.y;
    }
    if (i < n) {
        double2 x = a[i];
        acc0 += x.x * x.x + x.y * x.y;
    }
    double s = block_sum(acc0 + acc1);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedThreads) k_sum_partials(const double *partial, int np,
                                                              double *out) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += kRedThreads) acc += partial[i];
    double s = block_sum(acc);
    if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(kRedThreads) k_probs(const double2 *__restrict__ a, int64_t n,
                                                       double *__restrict__ p) {
    int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
    if (i < n) {
        double2 x = a[i];
        p[i] = __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y));
    }
}

// Qubit relabeling (layout.py:71-83): dst[p] = src[route(p)], route sending
// bit j of p to bit p2l[j].  Writes are coalesced; reads gather (coalesced
// whenever the low bits map to themselves).
struct BitMap {
    int8_t p2l[64];
};

__global__ void __launch_bounds__(kRedThreads) k_permute_bits(const double2 *__restrict__ src,
                                                              double2 *__restrict__ dst, int64_t n,
                                                              int nbits, BitMap m) {
    const int64_t p = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
    if (p >= n) return;
    int64_t s = 0;
    for (int j = 0; j < nbits; ++j) s |= ((p >> j) & 1) << m.p2l[j];
    dst[p] = src[s];
}

int launch_permute(const double2 *src, double2 *dst, int64_t n, const int *p2l, int nbits, cudaStream_t s) {
    BitMap m;
    for (int j = 0; j < 64; ++j) m.p2l[j] = (int8_t)(j < nbits ? p2l[j] : 0);
    int64_t blocks = (n + kRedThreads - 1) / kRedThreads;
    k_permute_bits<<<(unsigned)blocks, kRedThreads, 0, s>>>(src, dst, n, nbits, m);
    return 1;
}

// scratch: at least kRedBlocks + 1 doubles of device memory.
int launch_norm2(const double2 *a, int64_t n, double *scratch, cudaStream_t s) {
    int blocks = (int)((n + kRedThreads - 1) / kRedThreads);
    if (blocks > kRedBlocks) blocks = kRedBlocks;
    if (blocks < 1) blocks = 1;
    k_norm_partial<<<blocks, kRedThreads, 0, s>>>(a, n, scratch);
    k_sum_partials<<<1, kRedThreads, 0, s>>>(scratch, blocks, scratch + kRedBlocks);
    return 2;
}

int norm_scratch_doubles() { return kRedBlocks + 1; }

int launch_probs(const double2 *a, int64_t n, double *p, cudaStream_t s) {
    int64_t blocks = (n + kRedThreads - 1) / kRedThreads;
    k_probs<<<(unsigned)blocks, kRedThreads, 0, s>>>(a, n, p);
    return 1;
}

}  // namespace svb
