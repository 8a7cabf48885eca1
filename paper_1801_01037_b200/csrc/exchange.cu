// exchange.cu -- global-qubit (rank-bit) gate kernels.
//
// A gate whose target bit is a rank bit pairs local index j of rank r with
// local index j of partner r ^ 2^(t-(n-k)) (partition.py:126-137).
//
// k_exchange_own_row: the paper's single-amplitude protocol, batched: this
//   rank received the partner's amplitudes `other` and updates only its own
//   row (engine.py:249-254 scheme b; engine.py:257-272 chunked).  Used by the
//   multi-process engine after an NCCL send/recv of a chunk.
// k_pair_update: both rows of pairs (lo_slab[j], hi_slab[j]).  With peer
//   access one GPU reads the partner slab over NVLink and writes both
//   amplitudes back: the lower rank of a pair covers j < L/2, the upper rank
//   j >= L/2: each direction of the link carries 16*L bytes (a rank's reads
//   and writes of the partner's half, plus the partner's of its own) -- the
//   bytes of a slab exchange, but with no staging buffer, no send-back and
//   no separate update pass (the work split of scheme a, engine.py:206-238).
#include "svb_common.cuh"

namespace svb {

constexpr int kXThreads = 256;
constexpr int kXUpt = 4;

template <int KIND>
__global__ void __launch_bounds__(kXThreads) k_exchange_own_row(double2 *__restrict__ own,
                                                                const double2 *__restrict__ other,
                                                                int64_t count, Gate g, int own_is_low,
                                                                int cbit, int64_t offset) {
    const int64_t base = int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x;
    double2 mine[kXUpt], oth[kXUpt];
    bool on[kXUpt];
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        int64_t j = base + int64_t(k) * kXThreads;
        on[k] = j < count && (cbit < 0 || (((offset + j) >> cbit) & 1));
        if (on[k]) {
            mine[k] = own[j];
            oth[k] = other[j];
        }
    }
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        if (!on[k]) continue;
        int64_t j = base + int64_t(k) * kXThreads;
        own[j] = own_is_low ? row<KIND>(g, false, mine[k], oth[k]) : row<KIND>(g, true, oth[k], mine[k]);
    }
}

template <int KIND>
__global__ void __launch_bounds__(kXThreads) k_pair_update(double2 *lo_slab, double2 *hi_slab,
                                                           int64_t begin, int64_t end, Gate g,
                                                           int cbit) {
    const int64_t base = begin + int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x;
    double2 lo[kXUpt], hi[kXUpt];
    bool on[kXUpt];
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        int64_t j = base + int64_t(k) * kXThreads;
        on[k] = j < end && (cbit < 0 || ((j >> cbit) & 1));
        if (on[k]) {
            lo[k] = lo_slab[j];
            hi[k] = hi_slab[j];
        }
    }
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        if (!on[k]) continue;
        int64_t j = base + int64_t(k) * kXThreads;
        pair_both<KIND>(g, lo[k], hi[k]);
        lo_slab[j] = lo[k];
        hi_slab[j] = hi[k];
    }
    // peer stores are visible system-wide before the stream's next signal
    // (k_signal) can be observed by the partner
    __threadfence_system();
}

// Control-masked exchange (regime ii, engine.py:444-447): only local indices
// with bit cbit set take part.  Packed index p (offset + p) maps to local
// index insert_bit(offset + p, cbit, 1).
__global__ void __launch_bounds__(kXThreads) k_pack_ctrl(const double2 *__restrict__ src,
                                                         double2 *__restrict__ dst, int64_t count,
                                                         int cbit, int64_t offset) {
    const int64_t base = int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x;
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        int64_t p = base + int64_t(k) * kXThreads;
        if (p < count) dst[p] = src[insert_bit(offset + p, cbit, 1)];
    }
}

// Half-slab gather / scatter for a global<->local qubit swap: the elements
// whose local bit `bit` equals `value`, in index order (packed index p is
// local index insert_bit(offset + p, bit, value)).
__global__ void __launch_bounds__(kXThreads) k_pack_half(const double2 *__restrict__ src,
                                                         double2 *__restrict__ dst, int64_t count, int bit,
                                                         int value, int64_t offset) {
    const int64_t base = int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x;
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        int64_t p = base + int64_t(k) * kXThreads;
        if (p < count) dst[p] = src[insert_bit(offset + p, bit, value)];
    }
}

__global__ void __launch_bounds__(kXThreads) k_unpack_half(double2 *__restrict__ dst,
                                                           const double2 *__restrict__ src, int64_t count,
                                                           int bit, int value, int64_t offset) {
    const int64_t base = int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x;
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        int64_t p = base + int64_t(k) * kXThreads;
        if (p < count) dst[insert_bit(offset + p, bit, value)] = src[p];
    }
}

template <int KIND>
__global__ void __launch_bounds__(kXThreads) k_exchange_packed(double2 *__restrict__ own,
                                                               const double2 *__restrict__ other,
                                                               int64_t count, Gate g, int own_is_low,
                                                               int cbit, int64_t offset) {
    const int64_t base = int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x;
    double2 mine[kXUpt], oth[kXUpt];
    int64_t j[kXUpt];
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        int64_t p = base + int64_t(k) * kXThreads;
        j[k] = p < count ? insert_bit(offset + p, cbit, 1) : -1;
        if (j[k] >= 0) {
            mine[k] = own[j[k]];
            oth[k] = other[p];
        }
    }
#pragma unroll
    for (int k = 0; k < kXUpt; ++k) {
        if (j[k] < 0) continue;
        own[j[k]] = own_is_low ? row<KIND>(g, false, mine[k], oth[k]) : row<KIND>(g, true, oth[k], mine[k]);
    }
}

static unsigned grid_for(int64_t count) {
    return (unsigned)((count + int64_t(kXThreads) * kXUpt - 1) / (int64_t(kXThreads) * kXUpt));
}

LaunchInfo launch_exchange_own_row(double2 *own, const double2 *other, int64_t count, const Gate &g,
                                   int own_is_low, int cbit, int64_t offset, cudaStream_t s) {
    if (count <= 0) return LaunchInfo{0, PROF_EXCHANGE, 0};
    unsigned blocks = grid_for(count);
#define SVB_X(K) k_exchange_own_row<K><<<blocks, kXThreads, 0, s>>>(own, other, count, g, own_is_low, cbit, offset)
    switch (g.kind) {
        case K_REAL: SVB_X(K_REAL); break;
        case K_DIAG: SVB_X(K_DIAG); break;
        case K_ANTI: SVB_X(K_ANTI); break;
        case K_RX: SVB_X(K_RX); break;
        default: SVB_X(K_GENERAL); break;
    }
#undef SVB_X
    // own read + write, partner chunk read (control-masked: half of each)
    return LaunchInfo{1, PROF_EXCHANGE, (cbit >= 0 ? count / 2 : count) * 48};
}

LaunchInfo launch_pack_ctrl(const double2 *src, double2 *dst, int64_t count, int cbit, int64_t offset,
                            cudaStream_t s) {
    if (count <= 0) return LaunchInfo{0, PROF_EXCHANGE, 0};
    k_pack_ctrl<<<grid_for(count), kXThreads, 0, s>>>(src, dst, count, cbit, offset);
    return LaunchInfo{1, PROF_EXCHANGE, count * 32};
}

LaunchInfo launch_pack_half(const double2 *src, double2 *dst, int64_t count, int bit, int value, int64_t offset,
                            cudaStream_t s) {
    if (count <= 0) return LaunchInfo{0, PROF_EXCHANGE, 0};
    k_pack_half<<<grid_for(count), kXThreads, 0, s>>>(src, dst, count, bit, value, offset);
    return LaunchInfo{1, PROF_EXCHANGE, count * 32};
}

LaunchInfo launch_unpack_half(double2 *dst, const double2 *src, int64_t count, int bit, int value, int64_t offset,
                              cudaStream_t s) {
    if (count <= 0) return LaunchInfo{0, PROF_EXCHANGE, 0};
    k_unpack_half<<<grid_for(count), kXThreads, 0, s>>>(dst, src, count, bit, value, offset);
    return LaunchInfo{1, PROF_EXCHANGE, count * 32};
}

LaunchInfo launch_exchange_packed(double2 *own, const double2 *other, int64_t count, const Gate &g,
                                  int own_is_low, int cbit, int64_t offset, cudaStream_t s) {
    if (count <= 0) return LaunchInfo{0, PROF_EXCHANGE, 0};
    unsigned blocks = grid_for(count);
#define SVB_K(K) k_exchange_packed<K><<<blocks, kXThreads, 0, s>>>(own, other, count, g, own_is_low, cbit, offset)
    switch (g.kind) {
        case K_REAL: SVB_K(K_REAL); break;
        case K_DIAG: SVB_K(K_DIAG); break;
        case K_ANTI: SVB_K(K_ANTI); break;
        case K_RX: SVB_K(K_RX); break;
        default: SVB_K(K_GENERAL); break;
    }
#undef SVB_K
    return LaunchInfo{1, PROF_EXCHANGE, count * 48};
}

// k_peer_swap_half: the rank-bit <-> local-bit swap of the layout engine
// over peer memory.  Half index j in [begin, end) names position
// ins(j, bit, va) of slab a and ins(j, bit, vb) of slab b (ins: insert `v`
// as bit `bit` of j); the two amplitudes trade places.  The two ranks of a
// pair split the j range, each reading and writing the partner's slab
// through NVLink -- the pack / send / receive / unpack of the NCCL engine in
// one kernel, no staging.
__global__ void __launch_bounds__(kXThreads) k_peer_swap_half(double2 *a, double2 *b, int64_t begin, int64_t end,
                                                              int bit, int va, int vb) {
    const int64_t stride = int64_t(gridDim.x) * kXThreads;
    const int64_t low = (int64_t(1) << bit) - 1;
    for (int64_t j = begin + int64_t(blockIdx.x) * kXThreads + threadIdx.x; j < end; j += stride) {
        const int64_t hi = (j >> bit) << (bit + 1), lo = j & low;
        const int64_t ia = hi | (int64_t(va) << bit) | lo, ib = hi | (int64_t(vb) << bit) | lo;
        const double2 x = a[ia], y = b[ib];
        a[ia] = y;
        b[ib] = x;
    }
    __threadfence_system();
}

// Stream-ordered pairwise rank synchronisation of the peer transport (no
// host round trip): k_signal runs after every earlier kernel of its stream
// (whose peer stores each ended in a system fence) and publishes `value`
// into the partner's flag word with release semantics; the partner's stream
// waits on its own word with cuStreamWaitValue32 (>= value), a front-end
// wait that occupies no SM.
__global__ void k_signal(unsigned *flag, unsigned value) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

LaunchInfo launch_signal(unsigned *flag, unsigned value, cudaStream_t s) {
    k_signal<<<1, 1, 0, s>>>(flag, value);
    return LaunchInfo{1, PROF_SYNC, 0};
}

// SM-driven peer copy (link-ceiling probe): dst[i] = src[i], 16 B per
// element, four loads in flight per thread, grid-stride over 148 x 8 CTAs.
__global__ void __launch_bounds__(kXThreads) k_peer_copy(double2 *__restrict__ dst, const double2 *__restrict__ src,
                                                         int64_t count) {
    const int64_t stride = int64_t(gridDim.x) * kXThreads * kXUpt;
    for (int64_t base = int64_t(blockIdx.x) * kXThreads * kXUpt + threadIdx.x; base < count; base += stride) {
        double2 v[kXUpt];
#pragma unroll
        for (int k = 0; k < kXUpt; ++k) {
            const int64_t j = base + int64_t(k) * kXThreads;
            if (j < count) v[k] = src[j];
        }
#pragma unroll
        for (int k = 0; k < kXUpt; ++k) {
            const int64_t j = base + int64_t(k) * kXThreads;
            if (j < count) dst[j] = v[k];
        }
    }
}

LaunchInfo launch_peer_copy(double2 *dst, const double2 *src, int64_t count, cudaStream_t s) {
    if (count <= 0) return LaunchInfo{0, PROF_EXCHANGE, 0};
    const int64_t blocks = std::min<int64_t>((count + kXThreads * kXUpt - 1) / (kXThreads * kXUpt), 148 * 8);
    k_peer_copy<<<(unsigned)blocks, kXThreads, 0, s>>>(dst, src, count);
    return LaunchInfo{1, PROF_EXCHANGE, count * 32};
}

LaunchInfo launch_peer_swap_half(double2 *a, double2 *b, int64_t begin, int64_t end, int bit, int va, int vb,
                                 cudaStream_t s) {
    if (end <= begin) return LaunchInfo{0, PROF_EXCHANGE, 0};
    const int64_t blocks = std::min<int64_t>((end - begin + kXThreads - 1) / kXThreads, 148 * 8);
    k_peer_swap_half<<<(unsigned)blocks, kXThreads, 0, s>>>(a, b, begin, end, bit, va, vb);
    return LaunchInfo{1, PROF_EXCHANGE, (end - begin) * 64};
}

LaunchInfo launch_pair_update(double2 *lo_slab, double2 *hi_slab, int64_t begin, int64_t end,
                              const Gate &g, int cbit, cudaStream_t s) {
    if (end <= begin) return LaunchInfo{0, PROF_EXCHANGE, 0};
    unsigned blocks = grid_for(end - begin);
#define SVB_P(K) k_pair_update<K><<<blocks, kXThreads, 0, s>>>(lo_slab, hi_slab, begin, end, g, cbit)
    switch (g.kind) {
        case K_REAL: SVB_P(K_REAL); break;
        case K_DIAG: SVB_P(K_DIAG); break;
        case K_ANTI: SVB_P(K_ANTI); break;
        case K_RX: SVB_P(K_RX); break;
        default: SVB_P(K_GENERAL); break;
    }
#undef SVB_P
    return LaunchInfo{1, PROF_EXCHANGE, (cbit >= 0 ? (end - begin) / 2 : (end - begin)) * 64};
}

}  // namespace svb
