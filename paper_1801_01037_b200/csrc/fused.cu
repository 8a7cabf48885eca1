// fused.cu -- op-list execution with multi-gate HBM passes.
//
// run_circuit applies one gate per sweep over the state (engine.py:483-494,
// _stride_cy.pyx:24-90): 7,800 full read+write passes for the configs[1]
// circuit.  Here a host-side planner packs gates whose qubits fit in a set S
// of FM = 11 qubits into one pass; k_fused streams the state tile by tile --
// a tile is the 2^11 amplitudes sharing every bit outside S -- through
// shared memory and applies all gates of the pass before writing it back:
// one HBM read + one HBM write per pass instead of per gate.
//
//  * S always holds qubits 0..flow-1 (flow = 3 by default), so a tile is
//    2^(FM-flow) runs of 2^flow contiguous amplitudes and every global access
//    is a coalesced 16 B-per-lane cp.async (load) / store.
//  * Gates run in "register groups": each of the 128 threads of a CTA holds
//    16 amplitudes spanning 4 local bits (the group's slots).  Every
//    non-diagonal gate of a group targets a slot, so its pair updates are
//    register-to-register; a control bit needs no slot (it is a register mask
//    or a per-thread predicate); diagonal gates (Z S T Rz CP) need no pairing
//    at all.  Shared memory is read and written once per group.
//  * The other 7 local bits index threads through a per-group map chosen so
//    the 8 lanes of each LDS.128/STS.128 phase hit distinct 16 B bank groups
//    under the swizzle phys(l) = l ^ fold3(l >> 3).
//  * X / CNOT are bit permutations: deferred to the end of their group and
//    folded into the group's affine store map (exact, no arithmetic).  Z is
//    an in-place negation; everything else uses the exact single-gate
//    arithmetic of svb_common.cuh.  A strict-order plan is therefore
//    bit-identical to op-by-op application; the default plan may hoist a gate
//    over earlier gates on disjoint qubits (they commute) and agrees to a few
//    ulp.
//  * The first / last group of a pass moves its registers straight from / to
//    HBM when its thread map keeps lanes 0-7 on 128 B lines (direct groups).
//  * Four persistent CTAs per SM (32 KiB tile each, 16 warps): while some
//    stream their tile the others compute (measured best of FM 10-12 x
//    2-8 CTAs: FM=12 x 2 CTAs 31.2k, FM=11 x 4 CTAs 31.8k, FM=10 x 8 28.7k
//    gate applications/s on configs[1]).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <atomic>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/svb.h"
#include "svb_common.cuh"

namespace svb {

LaunchInfo launch_gate(double2 *a, int64_t n_amps, const Gate &g, int t, int c, cudaStream_t s);

}  // namespace svb
#include "fused_desc.h"
namespace svb {

// 16 B-granular XOR swizzle: bits 3-5, 6-8, 9-11, 12 fold into bits 0-2, so local
// bit j moves the 16 B chunk inside a 128 B line along axis (j mod 3).  It is
// linear over XOR, so swz(l0 | d) = swz(l0) ^ swz(d) for disjoint bits.
__host__ __device__ __forceinline__ int fold3(int x) { return (x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7; }
__host__ __device__ __forceinline__ int swz(int l) { return l ^ fold3(l >> 3); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// XOR of the per-slot offsets selected by the bits of register index i
template <class T, class S>
__device__ __forceinline__ T xcombo(const S *s, int i) {
    T r = 0;
#pragma unroll
    for (int k = 0; k < FSLOTS; ++k)
        if ((i >> k) & 1) r ^= (T)s[k];
    return r;
}

// x * u for u in {1, i, -1, -i} (code 0..3): exact, equal to the reference's
// (ac - bd, ad + bc) up to the sign of zero
__device__ __forceinline__ double2 unit_mul(int code, double2 x) {
    double2 r = (code & 1) ? make_double2(-x.y, x.x) : x;
    return (code & 2) ? make_double2(-r.x, -r.y) : r;
}

template <int KIND, int S, int CTRL, bool FMA>
__device__ __forceinline__ void nd_gate(double2 (&v)[FREGS], const FGate &fg) {
    const unsigned cm = fg.cmask;
    double2 q11 = make_double2(0, 0), q12 = q11, q21 = q11, q22 = q11;
    if (KIND != FK_X && KIND != FK_Y && KIND != FK_UANTI) {
        q11 = fg.m[0];
        q12 = fg.m[1];
        q21 = fg.m[2];
        q22 = fg.m[3];
    }
#pragma unroll
    for (int i = 0; i < FREGS; ++i) {
        if (i & (1 << S)) continue;
        if (CTRL && !((cm >> i) & 1)) continue;
        double2 &lo = v[i];
        double2 &hi = v[i | (1 << S)];
        const double2 t = lo;
        if (KIND == FK_X) {
            lo = hi;
            hi = t;
        } else if (KIND == FK_Y) {  // lo' = -i*hi, hi' = i*lo
            lo = make_double2(hi.y, -hi.x);
            hi = make_double2(-t.y, t.x);
        } else if (KIND == FK_UANTI) {
            lo = unit_mul(fg.u & 3, hi);
            hi = unit_mul((fg.u >> 2) & 3, t);
        } else if (KIND == FK_REAL) {
            if (FMA) pair_both_fma<K_REAL>(q11, q12, q21, q22, lo, hi); else pair_both_c<K_REAL>(q11, q12, q21, q22, lo, hi);
        } else if (KIND == FK_ANTI) {
            if (FMA) pair_both_fma<K_ANTI>(q11, q12, q21, q22, lo, hi); else pair_both_c<K_ANTI>(q11, q12, q21, q22, lo, hi);
        } else if (KIND == FK_RX) {
            if (FMA) pair_both_fma<K_RX>(q11, q12, q21, q22, lo, hi); else pair_both_c<K_RX>(q11, q12, q21, q22, lo, hi);
        } else {
            if (FMA) pair_both_fma<K_GENERAL>(q11, q12, q21, q22, lo, hi); else pair_both_c<K_GENERAL>(q11, q12, q21, q22, lo, hi);
        }
    }
}

template <int VAR, int TP, int CTRL, bool FMA>
__device__ __forceinline__ void diag_gate(double2 (&v)[FREGS], const FGate &fg, int l0) {
    const unsigned cm = fg.cmask;
    const double2 d0 = fg.m[0], d1 = fg.m[3];
    bool tb = false;
    if (TP == FSLOTS) {
        tb = (l0 >> fg.tl) & 1;
        if (VAR != FD_GENERAL && !tb) return;  // q11 == 1: the |0> half is untouched
    }
    const double2 f = (TP == FSLOTS && VAR == FD_GENERAL) ? (tb ? d1 : d0) : d1;
#pragma unroll
    for (int i = 0; i < FREGS; ++i) {
        if (CTRL && !((cm >> i) & 1)) continue;
        const bool b = TP == FSLOTS ? true : ((i >> TP) & 1);
        if (VAR != FD_GENERAL && !b) continue;
        double2 &x = v[i];
        if (VAR == FD_GENERAL) x = FMA ? cmul_f(TP == FSLOTS ? f : (b ? d1 : d0), x) : cmul(TP == FSLOTS ? f : (b ? d1 : d0), x);
        if (VAR == FD_D1) x = FMA ? cmul_f(f, x) : cmul(f, x);
        if (VAR == FD_Z) x = make_double2(-x.x, -x.y);
        if (VAR == FD_S) x = make_double2(-x.y, x.x);
        if (VAR == FD_SDG) x = make_double2(x.y, -x.x);
    }
}

#define SVB_OPND(K, S, C) (((K) * FSMAX + (S)) * 2 + (C))
#define SVB_OPDG(V, T, C) (FOP_DIAG + ((V) * (FSMAX + 1) + (T)) * 2 + (C))
#define SVB_ND2(K, S) \
    case SVB_OPND(K, S, 0): nd_gate<K, S, 0, FMA>(v, fg); break; \
    case SVB_OPND(K, S, 1): nd_gate<K, S, 1, FMA>(v, fg); break;
#if SVB_FSLOTS == 5
#define SVB_ND(K) SVB_ND2(K, 0) SVB_ND2(K, 1) SVB_ND2(K, 2) SVB_ND2(K, 3) SVB_ND2(K, 4)
#elif SVB_FSLOTS == 4
#define SVB_ND(K) SVB_ND2(K, 0) SVB_ND2(K, 1) SVB_ND2(K, 2) SVB_ND2(K, 3)
#else
#define SVB_ND(K) SVB_ND2(K, 0) SVB_ND2(K, 1) SVB_ND2(K, 2)
#endif
#define SVB_DG2(V, T) \
    case SVB_OPDG(V, T, 0): diag_gate<V, T, 0, FMA>(v, fg, l0); break; \
    case SVB_OPDG(V, T, 1): diag_gate<V, T, 1, FMA>(v, fg, l0); break;
// target on a thread bit: encoded tpos FTPOS_THREAD, the kernel's TP = FSLOTS
#define SVB_DGT(V) \
    case SVB_OPDG(V, FTPOS_THREAD, 0): diag_gate<V, FSLOTS, 0, FMA>(v, fg, l0); break; \
    case SVB_OPDG(V, FTPOS_THREAD, 1): diag_gate<V, FSLOTS, 1, FMA>(v, fg, l0); break;
#if SVB_FSLOTS == 5
#define SVB_DG(V) SVB_DG2(V, 0) SVB_DG2(V, 1) SVB_DG2(V, 2) SVB_DG2(V, 3) SVB_DG2(V, 4) SVB_DGT(V)
#elif SVB_FSLOTS == 4
#define SVB_DG(V) SVB_DG2(V, 0) SVB_DG2(V, 1) SVB_DG2(V, 2) SVB_DG2(V, 3) SVB_DGT(V)
#else
#define SVB_DG(V) SVB_DG2(V, 0) SVB_DG2(V, 1) SVB_DG2(V, 2) SVB_DGT(V)
#endif

// Register-permuting ops (X, Y, unit phases) as their own cases make every
// switch arm end with v[] in different physical registers, and ptxas then
// re-shuffles all 64 registers at the loop head on EVERY gate.  With
// SVB_FUSED_PERM_OPS 0 they run through the arithmetic arms instead (still
// exact: products with +-1 / +-i are exact).
#ifndef SVB_FUSED_PERM_OPS
#define SVB_FUSED_PERM_OPS 0
#endif
constexpr bool kPermOps = SVB_FUSED_PERM_OPS != 0;
// Fewer switch arms = smaller hot code: ncu showed 23 % of warp stalls as
// `no_instructions` (instruction fetch) with every (kind, slot, control) arm.
#ifndef SVB_COMPACT_DISPATCH
#define SVB_COMPACT_DISPATCH 1
#endif
constexpr bool kCompact = SVB_COMPACT_DISPATCH != 0;

template <bool FMA>
__device__ __forceinline__ void run_gate(double2 (&v)[FREGS], const FGate &fg, int l0, unsigned op) {
    switch (op) {
#if SVB_COMPACT_DISPATCH
        // controlled arithmetic gates all take the general arm (exact for every
        // matrix class); uncontrolled ones get their specialised arm
#define SVB_NDU(K, S) case SVB_OPND(K, S, 0): nd_gate<K, S, 0, FMA>(v, fg); break;
#define SVB_NDC(S) case SVB_OPND(FK_GENERAL, S, 1): nd_gate<FK_GENERAL, S, 1, FMA>(v, fg); break;
#if SVB_FSLOTS == 5
#define SVB_SLOTS(M, K) M(K, 0) M(K, 1) M(K, 2) M(K, 3) M(K, 4)
#elif SVB_FSLOTS == 4
#define SVB_SLOTS(M, K) M(K, 0) M(K, 1) M(K, 2) M(K, 3)
#else
#define SVB_SLOTS(M, K) M(K, 0) M(K, 1) M(K, 2)
#endif
#define SVB_NDC2(K, S) SVB_NDC(S)
        SVB_SLOTS(SVB_NDU, FK_GENERAL)
        SVB_SLOTS(SVB_NDU, FK_REAL)
        SVB_SLOTS(SVB_NDU, FK_ANTI)
        SVB_SLOTS(SVB_NDU, FK_RX)
        SVB_SLOTS(SVB_NDC2, 0)
#define SVB_DGU(V, T) case SVB_OPDG(V, T, 0): diag_gate<V, T, 0, FMA>(v, fg, l0); break;
        SVB_SLOTS(SVB_DGU, FD_Z)
        case SVB_OPDG(FD_Z, FTPOS_THREAD, 0): diag_gate<FD_Z, FSLOTS, 0, FMA>(v, fg, l0); break;
        SVB_DG(FD_GENERAL)
        SVB_DG(FD_D1)
        default: break;
    }
}
#else
        SVB_ND(FK_GENERAL)
        SVB_ND(FK_REAL)
        SVB_ND(FK_ANTI)
        SVB_ND(FK_RX)
#if SVB_FUSED_PERM_OPS
        SVB_ND(FK_UANTI)
        SVB_ND(FK_X)
        SVB_ND(FK_Y)
        SVB_DG(FD_S)
        SVB_DG(FD_SDG)
#endif
        SVB_DG(FD_Z)  // negation in place: no register renaming
        SVB_DG(FD_GENERAL)
        SVB_DG(FD_D1)
        default: break;
    }
}
#endif

template <bool FMA>
__global__ void __launch_bounds__(FTHREADS, FCTAS_PER_SM) k_fused(double2 *__restrict__ a, int64_t ntiles,
                                                                  const __grid_constant__ FPass P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *bufs = reinterpret_cast<double2 *>(smem_raw);
    int64_t *rowoff = reinterpret_cast<int64_t *>(smem_raw + kNBuf * FTILE * sizeof(double2));
    const int tid = threadIdx.x;
    const int flow = P.flow;
    const int nrows = FTILE >> flow;
    const int colmask = (1 << flow) - 1;
    for (int r = tid; r < nrows; r += FTHREADS) {
        int64_t off = 0;
        for (int j = 0; j < FM - flow; ++j)
            if ((r >> j) & 1) off |= int64_t(1) << P.rowbit[j];
        rowoff[r] = off;
    }
    __syncthreads();

    const int last = P.ngroups - 1;
    auto tile_base = [&](int64_t t) {
        int64_t b = 0;
        for (int j = 0; j < P.ncomp; ++j)
            if ((t >> j) & 1) b |= int64_t(1) << P.comp[j];
        return b;
    };
    auto fill = [&](double2 *dst, int64_t b) {
#pragma unroll
        for (int k = 0; k < FREGS; ++k) {
            int e = tid + k * FTHREADS;
            cp_async16(&dst[swz(e)], &a[b + rowoff[e >> flow] + (e & colmask)]);
        }
        cp_async_commit();
    };
    // double-buffered mode: tile i+1 streams into the other buffer while the
    // groups of tile i run (the first group then reads shared memory)
    const bool direct_first = P.direct_first && !kDB;
    if (kDB && blockIdx.x < ntiles) fill(bufs, tile_base(blockIdx.x));
    int it = 0;
    for (int64_t tix = blockIdx.x; tix < ntiles; tix += gridDim.x, ++it) {
        double2 *buf = bufs + (kDB ? (it & 1) * FTILE : 0);
        const int64_t base = tile_base(tix);
        if (kDB) {
            cp_async_wait_all();
            __syncthreads();
            const int64_t next = tix + gridDim.x;
            if (next < ntiles) fill(bufs + ((it + 1) & 1) * FTILE, tile_base(next));
        } else if (!direct_first) {
            fill(buf, base);
            cp_async_wait_all();
            __syncthreads();
        }

        unsigned char *sbytes = reinterpret_cast<unsigned char *>(buf);
        for (int gi = 0; gi < P.ngroups; ++gi) {
            const FGroup &G = P.groups[gi];
            double2 v[FREGS];
            if (gi == 0 && direct_first) {
                // first group straight from HBM: lanes 0-7 hold 8 consecutive
                // amplitudes (local bits 0-2), so each LDG.128 is 4 full 128 B lines
                // through the group's load map Q: offsets combine by XOR
                int64_t g0 = P.gl_b;
                unsigned tg = tid;
                asm volatile("" : "+r"(tg));
#pragma unroll
                for (int j = 0; j < FTBITS; ++j)
                    if ((tg >> j) & 1) g0 ^= P.gl_t[j];
#pragma unroll
                for (int i = 0; i < FREGS; ++i)
                    v[i] = __ldcs(a + (base | (g0 ^ xcombo<int64_t>(P.gl_s, i))));
            } else {
                // Shared-memory byte offset of register i: swizzle and the store
                // map are XOR-linear, so it is the XOR of host-precomputed per-bit
                // offsets: thread bits (ld_t) and slot bits (ld_s).
                unsigned a0 = G.ld_b, tg = tid;
                asm volatile("" : "+r"(tg));  // keep the per-bit masks out of the loop-invariant set
#pragma unroll
                for (int j = 0; j < FTBITS; ++j) a0 ^= (0u - ((tg >> j) & 1u)) & G.ld_t[j];
#pragma unroll
                for (int i = 0; i < FREGS; ++i) {
                    unsigned off = a0 ^ xcombo<unsigned>(G.ld_s, i);
                    v[i] = *reinterpret_cast<const double2 *>(sbytes + off);
                }
            }
            // gate header word (op | tl << 8 | cl << 16 | u << 24) is fetched one
            // gate ahead so the dispatch branch does not wait on the load
            const int qend = G.first + G.count;
            unsigned hdr = G.count > 0 ? *reinterpret_cast<const unsigned *>(&P.gates[G.first].op) : 0u;
            for (int q = G.first; q < qend; ++q) {
                const unsigned cur = hdr;
                if (q + 1 < qend) hdr = *reinterpret_cast<const unsigned *>(&P.gates[q + 1].op);
                const int cl = (int8_t)(cur >> 16);
                if (cl >= 0 && !((tid >> cl) & 1)) continue;  // thread-bit control clear
                run_gate<FMA>(v, P.gates[q], tid, cur & 0xffu);
            }
            if (gi == last && P.direct_last) {
                // last group straight to HBM through the store map P.  If this
                // group also loaded from HBM, a permuted store may hit an
                // address another thread has not read yet: barrier first
                // (bar.sync orders the block's earlier loads before later stores).
                if (G.perm && gi == 0 && direct_first) __syncthreads();
                int64_t g0 = P.gs_b;
                unsigned tg = tid;
                asm volatile("" : "+r"(tg));
#pragma unroll
                for (int j = 0; j < FTBITS; ++j)
                    if ((tg >> j) & 1) g0 ^= P.gs_t[j];
                // P mixes bits, so the per-register offset combines by XOR
                // with g0 (not by addition); tile bits stay disjoint (OR base)
#pragma unroll
                for (int i = 0; i < FREGS; ++i)
                    __stcs(a + (base | (g0 ^ xcombo<int64_t>(P.gs_s, i))),
                           v[i]);
                continue;
            }
            // Store register l at P(l) = M l ^ mb (identity unless the group
            // ends with X/CNOT gates); P is affine, so again an XOR of
            // per-bit offsets (st_b, st_t, st_s).  A permuted store writes
            // slots other threads loaded: wait for all loads first.
            if (G.perm) __syncthreads();
            unsigned b0 = G.st_b, ts = tid;
            asm volatile("" : "+r"(ts));
#pragma unroll
            for (int j = 0; j < FTBITS; ++j) b0 ^= (0u - ((ts >> j) & 1u)) & G.st_t[j];
#pragma unroll
            for (int i = 0; i < FREGS; ++i) {
                unsigned off = b0 ^ xcombo<unsigned>(G.st_s, i);
                *reinterpret_cast<double2 *>(sbytes + off) = v[i];
            }
            __syncthreads();
        }

        if (!P.direct_last) {
            int64_t base_s = base;  // recompute store addresses rather than keep 16 live
            asm volatile("" : "+l"(base_s));
#pragma unroll
            for (int k = 0; k < FREGS; ++k) {
                int e = tid + k * FTHREADS;
                a[base_s + rowoff[e >> flow] + (e & colmask)] = buf[swz(e)];
            }
        }
        if (!kDB) __syncthreads();  // buffer free for the next tile's loads
    }
    if (kDB) cp_async_wait_all();
}

// ---------------------------------------------------------------------------
// planner

struct PlanPass {
    uint64_t S = 0;  // global qubits in the tile
    uint64_t T = 0;  // targets of its non-diagonal ops
    std::vector<int> ops;
};

static int popc(uint64_t x) { return __builtin_popcountll(x); }

// 128 B runs (3 low qubits in every tile; 4 measured 1 % slower)
static int flow_bits() { return 3; }

// X/CNOT fold into the load / store maps (instead of the arithmetic arms)
static bool perm_fold() { return true; }

// direct HBM first/last groups are always on
static bool no_direct() { return false; }
// First / last groups move registers from / to HBM directly even when their
// lanes do not cover whole 128 B lines: a 32 B sector is then touched by
// two instructions and L2 merges them, which costs less than a shared-memory
// round trip (configs[1]: 82.2k -> 85.6k).
static bool direct_any() { return true; }

static uint64_t op_mask(const svb_op &o) {
    uint64_t m = uint64_t(1) << o.target;
    if (o.kind == 1) m |= uint64_t(1) << o.control;
    return m;
}

// Commutation classes for hoisting (non-strict planners).  On each qubit an
// op acts as Z-type (diagonal there: diagonal gates, and every control),
// X-type (a I + b X: X, Rx -- and CNOT on its target) or general.  Two ops
// whose factors on every shared qubit are both Z-type or both X-type commute
// exactly, so a later op may be hoisted over an unplaced earlier one unless
// some shared qubit mixes classes.  (Reordering changes rounding only: the
// non-strict modes promise 1e-12, strict order is bit-exact.)
struct Blocking {
    uint64_t z = 0, x = 0, g = 0;
    uint64_t all() const { return z | x | g; }
};
static bool commute_hoist() { return true; }
static Blocking op_class(const svb_op &o) {
    Blocking b;
    const Gate g = make_gate(o.q);
    const uint64_t t = uint64_t(1) << o.target;
    const bool xtype = g.m[0].x == g.m[3].x && g.m[0].y == g.m[3].y && g.m[1].x == g.m[2].x &&
                       g.m[1].y == g.m[2].y;
    if (!commute_hoist())
        b.g = t;
    else if (g.kind == K_DIAG)
        b.z = t;
    else if (xtype)
        b.x = t;
    else
        b.g = t;
    if (o.kind == 1) {
        if (commute_hoist())
            b.z |= uint64_t(1) << o.control;
        else
            b.g |= uint64_t(1) << o.control;
    }
    return b;
}
// may op (class c) move ahead of the unplaced ops summarised in blk?
static bool hoistable(const Blocking &c, const Blocking &blk) {
    return (c.z & (blk.x | blk.g)) == 0 && (c.x & (blk.z | blk.g)) == 0 && (c.g & blk.all()) == 0;
}
static void block_add(Blocking &blk, const Blocking &c) {
    blk.z |= c.z;
    blk.x |= c.x;
    blk.g |= c.g;
}

// Greedy pass construction.  strict: only contiguous runs of ops.  Otherwise
// a scan over the remaining ops that hoists an op past skipped ones only if
// it shares no qubit with any skipped op (so every qubit keeps its order).
static int planner_kind() { return 3; }  // 1 greedy, 2 lookahead (async JIT's quick plan), 3 two-pass lookahead

// Lookahead pass construction (non-strict): grow the pass's qubit set S one
// gate's qubits at a time, choosing among the ready gates the one whose new
// qubits admit the most gates per new qubit; after every growth, absorb every
// ready gate whose qubits are already in S.  Gate order per qubit is kept by
// the same blocked-qubit scan as the greedy planner.
static std::vector<PlanPass> plan_lookahead(int n, const svb_op *ops, int nops, int fm) {
    std::vector<PlanPass> passes;
    const uint64_t low = (uint64_t(1) << flow_bits()) - 1;
    std::vector<char> done(nops, 0);
    std::vector<Blocking> cls(nops);
    for (int i = 0; i < nops; ++i) cls[i] = op_class(ops[i]);
    int first = 0;
    const int window = 1024;
    std::vector<int> taken;
    // ops that can join a pass with qubit set S (without marking them)
    auto absorb_count = [&](uint64_t S, int lim) {
        Blocking blocked;
        int cnt = 0;
        for (int i = first; i < nops && i < first + window; ++i) {
            if (done[i]) continue;
            uint64_t m = op_mask(ops[i]);
            if (hoistable(cls[i], blocked) && (m & ~S) == 0) {
                if (++cnt >= lim) break;
            } else {
                block_add(blocked, cls[i]);
            }
        }
        return cnt;
    };
    while (first < nops) {
        PlanPass p;
        p.S = low;
        for (;;) {
            // absorb everything that fits S
            Blocking blocked;
            for (int i = first; i < nops && i < first + window && (int)p.ops.size() < FMAXG; ++i) {
                if (done[i]) continue;
                uint64_t m = op_mask(ops[i]);
                if (hoistable(cls[i], blocked) && (m & ~p.S) == 0) {
                    p.ops.push_back(i);
                    done[i] = 1;
                } else {
                    block_add(blocked, cls[i]);
                }
            }
            if (popc(p.S) >= fm || (int)p.ops.size() >= FMAXG) break;
            // candidate growths: ready gates needing new qubits that still fit
            uint64_t best = 0;
            double best_score = -1.0;
            int cands = 0;
            blocked = Blocking();
            for (int i = first; i < nops && i < first + window && cands < 24; ++i) {
                if (done[i]) continue;
                uint64_t m = op_mask(ops[i]);
                uint64_t add = m & ~p.S;
                if (hoistable(cls[i], blocked) && add && popc(p.S | m) <= fm) {
                    ++cands;
                    int gain = absorb_count(p.S | m, FMAXG);
                    double score = double(gain) / popc(add);
                    if (score > best_score) {
                        best_score = score;
                        best = m;
                    }
                }
                block_add(blocked, cls[i]);
            }
            if (!best) break;
            p.S |= best;
        }
        while (first < nops && done[first]) ++first;
        if (p.ops.empty()) {  // cannot happen (the first pending op always fits) -- guard
            p.ops.push_back(first);
            p.S |= op_mask(ops[first]);
            done[first] = 1;
            while (first < nops && done[first]) ++first;
        }
        for (int q = 0; q < n && popc(p.S) < fm; ++q) p.S |= uint64_t(1) << q;
        passes.push_back(std::move(p));
    }
    return passes;
}

// Two-pass lookahead over the lookahead planner: for each pass, try each
// candidate first growth of S (the ready gates that bring new qubits), finish
// that pass greedily, then plan the following pass greedily too, and keep the
// first growth that retires the most ops over both passes.  Host-only and
// run once per circuit (compiled plans are cached).
static bool rotate_low() { return true; }  // (fixed low qubits measured 203 vs 171 passes)

// Qubits a pass need not tile (outside = true, runtime-specialised passes
// only): an op acts on each of its qubits as Z-type (diagonal there -- a
// diagonal gate's target, every control) or not.  A Z-type qubit outside the
// tile's set S is constant over a tile, so the op becomes a tile-uniform
// predicate (control) or a per-tile factor (diagonal target) and only its
// non-diagonal target must lie in S.  Within a pass every op touching a
// qubit outside S acts Z-type on it, so those ops commute there.
static uint64_t need_mask(const svb_op &o, bool outside) {
    if (!outside) return op_mask(o);
    return make_gate(o.q).kind == K_DIAG ? 0 : uint64_t(1) << o.target;
}

static std::vector<PlanPass> plan_beam(int n, const svb_op *ops, int nops, int fm, bool outside) {
    std::vector<PlanPass> passes;
    const uint64_t low = (uint64_t(1) << flow_bits()) - 1;
    const int nlow = flow_bits();
    // rotate: the qubits at physical bits 0..flow-1 change from pass to pass
    // (a pass's store may move any of its qubits there), so a pass needs only
    // nlow qubits of the previous pass's set -- not nlow fixed qubits
    const bool rotate = rotate_low();
    uint64_t anchor = low;  // the set S must share >= nlow qubits with
    auto room = [&](uint64_t S) {  // tile bits S needs once topped up from the anchor
        return popc(S) + std::max(0, nlow - popc(S & anchor));
    };
    std::vector<Blocking> cls(nops);
    std::vector<uint64_t> tgt(nops);  // non-diagonal target bit (0 for diagonal ops)
    for (int i = 0; i < nops; ++i) {
        cls[i] = op_class(ops[i]);
        tgt[i] = make_gate(ops[i].q).kind == K_DIAG ? 0 : uint64_t(1) << ops[i].target;
    }
    std::vector<uint64_t> need(nops);  // qubits op i needs in the tile
    for (int i = 0; i < nops; ++i) need[i] = need_mask(ops[i], outside);
    const int tcap = 64;  // distinct non-diagonal targets per pass: no cap (caps measured slower)
    const int window = 1024;
    auto absorb = [&](std::vector<char> &done, int first, PlanPass &p, bool mark) {
        Blocking blocked;
        int cnt = 0;
        uint64_t T = p.T;
        for (int i = first; i < nops && i < first + window && (int)p.ops.size() + cnt < FMAXG; ++i) {
            if (done[i]) continue;
            uint64_t m = need[i];
            const bool tfit = !(tgt[i] & ~T) || popc(T) < tcap;
            if (hoistable(cls[i], blocked) && (m & ~p.S) == 0 && tfit) {
                T |= tgt[i];
                if (mark) {
                    p.ops.push_back(i);
                    done[i] = 1;
                } else {
                    ++cnt;
                }
            } else {
                block_add(blocked, cls[i]);
            }
        }
        if (mark) p.T = T;
        return cnt;
    };
    // candidate growths of p.S (distinct op masks, ready, fitting)
    auto candidates = [&](const std::vector<char> &done, int first, const PlanPass &p, int lim) {
        std::vector<uint64_t> out;
        Blocking blocked;
        for (int i = first; i < nops && i < first + window && (int)out.size() < lim; ++i) {
            if (done[i]) continue;
            uint64_t m = need[i];
            uint64_t add = m & ~p.S;
            if (hoistable(cls[i], blocked) && add && room(p.S | m) <= fm &&
                std::find(out.begin(), out.end(), m) == out.end())
                out.push_back(m);
            block_add(blocked, cls[i]);
        }
        return out;
    };
    // greedy pass (as plan_lookahead) from `first`, optionally forcing the first growth
    auto greedy = [&](std::vector<char> &done, int first, uint64_t forced) {
        PlanPass p;
        p.S = rotate ? 0 : low;
        bool forced_used = forced == 0;
        for (;;) {
            absorb(done, first, p, true);
            if (room(p.S) >= fm || (int)p.ops.size() >= FMAXG) break;
            uint64_t best = 0;
            if (!forced_used) {
                best = forced;
                forced_used = true;
            } else {
                double best_score = -1.0;
                for (uint64_t m : candidates(done, first, p, 24)) {
                    PlanPass q;
                    q.S = p.S | m;
                    int gain = absorb(done, first, q, false);
                    double score = double(gain) / popc(m & ~p.S);
                    if (score > best_score) {
                        best_score = score;
                        best = m;
                    }
                }
            }
            if (!best) break;
            p.S |= best;
        }
        return p;
    };
    std::vector<char> done(nops, 0);
    int first = 0;
    auto advance = [&](const std::vector<char> &d, int f) {
        while (f < nops && d[f]) ++f;
        return f;
    };
    while (first < nops) {
        // candidate first growths after the free absorb at S = low
        std::vector<char> d0 = done;
        PlanPass p0;
        p0.S = rotate ? 0 : low;
        absorb(d0, first, p0, true);
        const int ncand = 12, wa = 2, depth = 3;  // candidates, first-pass weight, passes looked at
        std::vector<uint64_t> cands = candidates(d0, first, p0, ncand);
        // candidates are scored independently (each on its own copy of
        // `done`), on up to 16 host threads; the first best in candidate
        // order wins, so the plan does not depend on the thread count
        std::vector<long> scores(cands.size(), -1);
        auto score_one = [&](size_t c) {
            std::vector<char> d1 = done;
            PlanPass a = greedy(d1, first, cands[c]);
            long score = wa * (long)a.ops.size();
            int f1 = first;
            for (int k = 1; k < depth; ++k) {
                f1 = advance(d1, f1);
                if (f1 >= nops) break;
                score += (long)greedy(d1, f1, 0).ops.size();
            }
            scores[c] = score;
        };
        const unsigned nthr = std::min<unsigned>((unsigned)cands.size(),
                                                 std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
        if (nthr > 1 && nops - first > 256) {
            std::atomic<size_t> next{0};
            std::vector<std::thread> pool;
            for (unsigned t = 1; t < nthr; ++t)
                pool.emplace_back([&] {
                    for (size_t c; (c = next++) < cands.size();) score_one(c);
                });
            for (size_t c; (c = next++) < cands.size();) score_one(c);
            for (auto &t : pool) t.join();
        } else {
            for (size_t c = 0; c < cands.size(); ++c) score_one(c);
        }
        uint64_t best_m = 0;
        long best_score = -1;
        for (size_t c = 0; c < cands.size(); ++c)
            if (scores[c] > best_score) {
                best_score = scores[c];
                best_m = cands[c];
            }
        PlanPass p = greedy(done, first, best_m);
        if (p.ops.empty()) {  // guard: the first pending op always fits
            p.ops.push_back(first);
            p.S |= op_mask(ops[first]);
            done[first] = 1;
        }
        first = advance(done, first);
        // top up: anchor qubits first (at least nlow of them), then any
        for (int q = 0; q < n && popc(p.S & anchor) < nlow; ++q)
            if ((anchor >> q) & 1) p.S |= uint64_t(1) << q;
        for (int q = 0; q < n && popc(p.S) < fm; ++q) p.S |= uint64_t(1) << q;
        if (rotate) anchor = p.S;
        passes.push_back(std::move(p));
    }
    return passes;
}

static std::vector<PlanPass> plan(int n, const svb_op *ops, int nops, bool strict, int fm, bool outside,
                                  int kind) {
    if (!strict && kind == 3) return plan_beam(n, ops, nops, fm, outside);
    if (!strict && kind == 2) return plan_lookahead(n, ops, nops, fm);
    std::vector<PlanPass> passes;
    const uint64_t low = (uint64_t(1) << flow_bits()) - 1;
    const uint64_t all = n >= 64 ? ~uint64_t(0) : ((uint64_t(1) << n) - 1);
    std::vector<char> done(nops, 0);
    int first = 0;
    const int window = 8192;
    while (first < nops) {
        PlanPass p;
        p.S = low;
        uint64_t blocked = 0;
        for (int i = first; i < nops && i < first + window; ++i) {
            if (done[i]) continue;
            uint64_t m = op_mask(ops[i]);
            bool fits = (m & blocked) == 0 && popc(p.S | m) <= fm && (int)p.ops.size() < FMAXG;
            if (fits) {
                p.S |= m;
                p.ops.push_back(i);
                done[i] = 1;
            } else {
                if (strict) break;
                blocked |= m;
                if ((blocked | p.S) == all && popc(p.S) == fm) {
                    // nothing outside S can join and every S qubit is blocked or
                    // free; keep scanning only while S-internal ops remain possible
                    if ((blocked & p.S) == p.S) break;
                }
            }
        }
        while (first < nops && done[first]) ++first;
        for (int q = 0; q < n && popc(p.S) < fm; ++q) p.S |= uint64_t(1) << q;
        passes.push_back(std::move(p));
    }
    return passes;
}

static int unit_code(double2 z) {
    if (z.x == 1.0 && z.y == 0.0) return 0;
    if (z.x == 0.0 && z.y == 1.0) return 1;
    if (z.x == -1.0 && z.y == 0.0) return 2;
    if (z.x == 0.0 && z.y == -1.0) return 3;
    return -1;
}

// registers (0..2^fs-1) whose slot-s bit is set
static unsigned slot_pattern(int s, int fs = FSLOTS) {
    unsigned m = 0;
    for (int i = 0; i < (1 << fs); ++i)
        if ((i >> s) & 1) m |= 1u << i;
    return m;
}

struct GateMeta {
    Gate g;
    int tl, cl;  // local bits (cl = -1: none, or outside the tile)
    int tt, ct;  // tile-index bits of a diagonal target / a control outside the tile (-1: none)
    bool diag;
    bool perm;
};

// Thread-bit -> local-bit map for a group: the 3 lowest thread bits (which
// vary across the 8 lanes of an LDS.128 phase) go to non-slot local bits
// with distinct (bit mod 3) so the swizzle spreads them over 8 chunks.
// pref: 3 local bits for lanes 0-2 that make a direct HBM side coalesced
// (nullptr: none); they win over bank-conflict freedom on the other side.
static void thread_map(int fm, int fs, const int *slots, int8_t *tmap, const int16_t *qcol = nullptr,
                       const int16_t *mcol = nullptr, bool need_ld = false, bool need_st = false,
                       const int *pref = nullptr) {
    bool is_slot[FMMAX] = {};
    for (int i = 0; i < fs; ++i) is_slot[slots[i]] = true;
    std::vector<int> free_bits;
    for (int b = 0; b < fm; ++b)
        if (!is_slot[b]) free_bits.push_back(b);
    int pick[3] = {-1, -1, -1};
    for (int r = 0; r < 3; ++r)
        for (int b : free_bits)
            if (b % 3 == r) {
                pick[r] = b;
                break;
            }
    std::vector<int> order;
    if (pick[0] >= 0 && pick[1] >= 0 && pick[2] >= 0) {
        order = {pick[0], pick[1], pick[2]};
        std::sort(order.begin(), order.end());
    }
    // With X/CNOT maps folded into the group's load (Q) or store (P) map, the
    // lanes of a phase address Q(l) / P(l) instead of l: keep the 3 lanes'
    // bank vectors independent for the accesses that go through shared
    // memory, otherwise each STS.128 / LDS.128 takes 2-4x the wavefronts.
    auto bank = [](int col) { return (col ^ (col >> 3) ^ (col >> 6) ^ (col >> 9) ^ (col >> 12)) & 7; };
    // wavefronts of one 8-lane phase whose lanes vary bits a, b, c through cols
    auto ways = [&](const int16_t *cols, int a, int b, int c) {
        int seen[8] = {0}, w = 0;
        for (int l = 0; l < 8; ++l) {
            int x = ((l & 1) ? bank(cols[a]) : 0) ^ ((l & 2) ? bank(cols[b]) : 0) ^ ((l & 4) ? bank(cols[c]) : 0);
            w = std::max(w, ++seen[x]);
        }
        return w;
    };
    auto cost = [&](int a, int b, int c) {
        return (need_ld ? ways(qcol, a, b, c) : 1) + (need_st ? ways(mcol, a, b, c) : 1);
    };
    if (pref) order = {pref[0], pref[1], pref[2]};
    if (qcol && !pref && (order.size() < 3 || cost(order[0], order[1], order[2]) > 2)) {
        const int nf = (int)free_bits.size();
        int best = order.size() == 3 ? cost(order[0], order[1], order[2]) : 1 << 20;
        for (int i = 0; i < nf && best > 2; ++i)
            for (int j = i + 1; j < nf && best > 2; ++j)
                for (int k = j + 1; k < nf && best > 2; ++k) {
                    const int c = cost(free_bits[i], free_bits[j], free_bits[k]);
                    if (c < best) {
                        best = c;
                        order = {free_bits[i], free_bits[j], free_bits[k]};
                    }
                }
    }
    for (int b : free_bits)
        if (std::find(order.begin(), order.end(), b) == order.end()) order.push_back(b);
    for (int j = 0; j < fm - fs; ++j) tmap[j] = (int8_t)order[j];
}

// In-register X / CNOT (see the group scan) pays off when passes are JIT
// compiled (a register rename); the interpreter would run them as arithmetic,
// so it keeps deferring them.  SVB_FUSE_REGPERM=0/1 forces either.
// (read per call: tests flip it to compare JIT and interpreter on one plan)
static bool reg_perm(unsigned flags) {
    const char *e = getenv("SVB_FUSE_REGPERM");
    return e ? atoi(e) != 0 : (flags & SVB_RUN_JIT) != 0;
}

static bool reg_perm_any_ctl() { return true; }

// (choosing each register group's slot set by a dry-run lookahead instead of
// first come was measured: configs[1] 544 -> 535 groups for twice the
// planning time and no speedup; off)
static bool group_lookahead() { return false; }

// Build the kernel descriptor for one pass; false if it does not fit.
// Qubit layout: logical qubit q lives at physical index bit phys[q] (nullptr:
// identity).  A pass tiles over the physical bits of its qubit set S -- which
// must include physical bits 0..flow-1 (whole 2^flow-amplitude rows) -- and
// may leave the state in a new layout phys_next that differs only inside S:
// its last group then stores every register through the extra bit
// permutation.  Gates name logical qubits; everything on the device is
// physical.
static bool defer_diag() { return true; }

static bool build_pass(int n, const svb_op *ops, const PlanPass &pp, FPass &P, bool strict, bool regperm,
                       int fm, const int8_t *phys = nullptr, const int8_t *phys_next = nullptr,
                       int fs = FSLOTS) {
    memset(&P, 0, sizeof(P));
    P.flow = flow_bits();
    P.fm = fm;
    P.fs = fs;
    const int tbits = fm - fs;
    auto ph = [&](int q) { return phys ? (int)phys[q] : q; };
    auto phn = [&](int q) { return phys_next ? (int)phys_next[q] : ph(q); };
    int local_of[64];
    int glob_of[FMMAX];  // local bit -> physical bit
    {
        std::vector<std::pair<int, int>> pq;  // (physical bit, logical qubit) of the tile
        for (int q = 0; q < n; ++q)
            if ((pp.S >> q) & 1) pq.push_back({ph(q), q});
        if ((int)pq.size() != fm) return false;
        std::sort(pq.begin(), pq.end());
        for (int j = 0; j < P.flow; ++j)
            if (pq[j].first != j) return false;  // rows must be physical bits 0..flow-1
        uint64_t tile_phys = 0;
        for (int q = 0; q < n; ++q) local_of[q] = -1;
        for (int j = 0; j < fm; ++j) {
            local_of[pq[j].second] = j;
            glob_of[j] = pq[j].first;
            tile_phys |= uint64_t(1) << pq[j].first;
            if (j >= P.flow) P.rowbit[j - P.flow] = (int8_t)pq[j].first;
        }
        int nc = 0;
        for (int b = 0; b < n; ++b)
            if (!((tile_phys >> b) & 1)) P.comp[nc++] = (int8_t)b;
        P.ncomp = nc;
    }
    // tile-index bit holding logical qubit q (q outside the tile)
    auto tile_bit = [&](int q) {
        for (int j = 0; j < P.ncomp; ++j)
            if (P.comp[j] == ph(q)) return j;
        return -1;
    };
    // store remap: old local bit of q -> local bit of phn(q) among the same physical bits
    int sig[FMMAX];
    bool remap = false;
    for (int q = 0; q < n; ++q) {
        if (local_of[q] < 0) continue;
        int r = 0;
        while (r < fm && glob_of[r] != phn(q)) ++r;
        if (r == fm) return false;  // phys_next must permute the tile's own bits
        sig[local_of[q]] = r;
        remap |= r != local_of[q];
    }
    if ((int)pp.ops.size() > FMAXG) return false;
    std::vector<GateMeta> meta;
    for (int oi : pp.ops) {
        const svb_op &o = ops[oi];
        GateMeta m;
        m.g = make_gate(o.q);
        m.tl = local_of[o.target];
        m.cl = o.kind == 1 ? local_of[o.control] : -1;
        m.diag = m.g.kind == K_DIAG;
        // Z-type qubits outside the tile (need_mask): tile-uniform predicates
        m.tt = m.tl < 0 ? tile_bit(o.target) : -1;
        m.ct = (o.kind == 1 && m.cl < 0) ? tile_bit(o.control) : -1;
        if (m.tl < 0 && !m.diag) return false;  // a non-diagonal target must be tiled
        if (m.tt >= 32 || m.ct >= 32) return false;
        // X and CNOT are bit permutations: folded into the group's store map
        // (a CNOT controlled from outside the tile differs per tile: it runs as
        // a predicated gate instead)
        m.perm = perm_fold() && m.g.kind == K_ANTI && unit_code(m.g.m[1]) == 0 &&
                 unit_code(m.g.m[2]) == 0 && m.ct < 0;
        meta.push_back(m);
    }
    // Order gates into register groups.  A group holds at most 4 target slots
    // of arithmetic gates; its X/CNOT gates are deferred to the group's end
    // (applied by the store map), which is exact because a pure permutation
    // commutes with every gate on other qubits -- so once a permutation is
    // deferred, later gates sharing its qubits wait for the next group.
    // strict: pass order, cut at a 5th slot or a permutation conflict.
    // Otherwise: repeated scans taking every ready gate (all earlier gates on
    // its qubits already placed) that fits.
    const int ng = (int)meta.size();
    struct GroupPlan {
        std::vector<int> gates;  // indices into meta, execution order (no perms)
        std::vector<int> slots;
        int mcol[FMMAX];         // post map P (store)
        int mb = 0;
        uint64_t permq = 0;
        int qcol[FMMAX];         // pre map Q (load): register l reads position Q(l)
        int qb = 0;
    };
    std::vector<GroupPlan> gps;
    auto new_group = [&]() {
        GroupPlan g;
        for (int j = 0; j < fm; ++j) g.mcol[j] = g.qcol[j] = 1 << j;
        gps.push_back(g);
        return &gps.back();
    };
    // A permutation C met before any arithmetic gate of the group is folded
    // into the load map instead: the state after C holds at l what was at
    // C(l) (C is an involution), so Q <- Q o C; no qubit gets blocked.
    auto pre_perm = [&](GroupPlan &g, const GateMeta &m) {
        if (m.cl >= 0) g.qcol[m.cl] ^= g.qcol[m.tl];  // CNOT: column c of (M_Q L_C)
        else g.qb ^= g.qcol[m.tl];                   // X: offset M_Q e_t
    };
    auto defer_perm = [&](GroupPlan &g, const GateMeta &m) {
        // compose C(x) = x ^ (x_c << t) (X: c = -1, always) after the current map
        auto C = [&](int x) { return (m.cl < 0 || ((x >> m.cl) & 1)) ? x ^ (1 << m.tl) : x; };
        auto Cl = [&](int x) { return (m.cl >= 0 && ((x >> m.cl) & 1)) ? x ^ (1 << m.tl) : x; };
        for (int j = 0; j < fm; ++j) g.mcol[j] = Cl(g.mcol[j]);
        g.mb = C(g.mb);
        g.permq |= (uint64_t(1) << m.tl) | (m.cl >= 0 ? uint64_t(1) << m.cl : 0);
    };
    auto gbits = [&](const GateMeta &m) {  // local bits only
        return (m.tl >= 0 ? uint64_t(1) << m.tl : 0) | (m.cl >= 0 ? uint64_t(1) << m.cl : 0);
    };
    // allowed: the group's slot set when chosen up front (0: first come)
    auto fits = [&](const GroupPlan &g, const GateMeta &m, bool first, uint64_t allowed) {
        if (m.diag) return true;
        // the first group keeps local bits 0-2 out of its slots so it can load
        // straight from HBM with coalesced 128 B lines (direct_first)
        if (!strict && first && m.tl < 3) return false;
        if (allowed) return ((allowed >> m.tl) & 1) != 0;
        return std::find(g.slots.begin(), g.slots.end(), m.tl) != g.slots.end() ||
               (int)g.slots.size() < fs;
    };
    auto take = [&](GroupPlan &g, int q, bool inreg = false) {
        const GateMeta &m = meta[q];
        if (m.perm && !inreg) {
            if (g.gates.empty() && g.permq == 0)
                pre_perm(g, m);
            else
                defer_perm(g, m);
            return;
        }
        if (!m.diag && std::find(g.slots.begin(), g.slots.end(), m.tl) == g.slots.end()) g.slots.push_back(m.tl);
        g.gates.push_back(q);
    };
    if (strict) {
        GroupPlan *g = new_group();
        for (int q = 0; q < ng; ++q) {
            const GateMeta &m = meta[q];
            bool ok = m.perm || ((gbits(m) & g->permq) == 0 && fits(*g, m, gps.size() == 1, 0));
            if (!ok) g = new_group();
            take(*g, q);
        }
    } else {
        std::vector<char> placed(ng, 0);
        int left = ng;
        // Fill group g from the unplaced gates: repeated scans taking every
        // ready gate (no earlier unplaced gate on its qubits) that fits.
        // mode 0: arithmetic only; 1: permutations too (post map);
        // 2: permutations only -- run first, they fold into the load map.
        auto fill_group = [&](GroupPlan &g, std::vector<char> &pl, int &lft, bool first, uint64_t allowed) {
            int taken = 0;
            auto scan = [&](int mode) {
                bool progress = false;
                uint64_t blocked = 0;  // local bits touched by an unplaced earlier gate
                for (int q = 0; q < ng; ++q) {
                    if (pl[q]) continue;
                    const GateMeta &m = meta[q];
                    const uint64_t bits = gbits(m);
                    // an X / CNOT whose target fits the group's slots runs in
                    // registers (a masked register swap) instead of being
                    // deferred to the store map, so it blocks nothing
                    // (also with a thread-bit control: a per-thread conditional swap)
                    const bool ctl_ok = m.cl < 0 || reg_perm_any_ctl() ||
                                        std::find(g.slots.begin(), g.slots.end(), m.cl) != g.slots.end();
                    const bool inreg = m.perm && mode == 0 && regperm && ctl_ok && (bits & blocked) == 0 &&
                                       (bits & g.permq) == 0 && fits(g, m, first, allowed);
                    bool ok = (bits & blocked) == 0 &&
                              (m.perm ? (mode != 0 || inreg)
                                      : (mode != 2 && (bits & g.permq) == 0 && fits(g, m, first, allowed)));
                    // a CNOT between local bits 0-2 and the rest, folded into the
                    // first group's load map, would break its coalesced HBM rows
                    if (mode == 2 && first && (bits & 7) && (bits & ~uint64_t(7))) ok = false;
                    if (ok) {
                        take(g, q, inreg);
                        pl[q] = 1;
                        --lft;
                        ++taken;
                        progress = true;
                    } else {
                        blocked |= bits;
                    }
                }
                return progress;
            };
            while (scan(2)) {
            }
            for (;;) {
                while (scan(0)) {
                }
                if (!scan(1)) break;
            }
            return taken;
        };
        auto fresh = [&]() {
            GroupPlan g;
            for (int j = 0; j < fm; ++j) g.mcol[j] = g.qcol[j] = 1 << j;
            return g;
        };
        while (left > 0) {
            const bool first = gps.empty();
            // Choose the slot set up front: grow it one local bit at a time,
            // each time the bit whose addition lets the group take the most
            // gates (a dry run of the same scans); stop when no bit helps.
            uint64_t allowed = 0;
            if (group_lookahead()) {
                int have = -1;
                for (int k = 0; k < fs; ++k) {
                    int best = have, bb = -1;
                    for (int b = 0; b < fm; ++b) {
                        if ((allowed >> b) & 1) continue;
                        if (first && b < 3) continue;
                        std::vector<char> pl = placed;
                        int lft = left;
                        GroupPlan tmp = fresh();
                        const int c = fill_group(tmp, pl, lft, first, allowed | (uint64_t(1) << b));
                        if (c > best) {
                            best = c;
                            bb = b;
                        }
                    }
                    if (bb < 0) break;
                    allowed |= uint64_t(1) << bb;
                    have = best;
                }
            }
            GroupPlan *g = new_group();
            fill_group(*g, placed, left, first, allowed);
            if (g->gates.empty() && g->permq == 0 && g->qb == 0 && allowed) {
                // (nothing fit the chosen set -- cannot happen, but never loop)
                fill_group(*g, placed, left, first, 0);
            }
        }
    }
    // Move diagonal gates to the latest group they commute into (no
    // non-diagonal gate or load / store permutation on their local bits in
    // between): diagonals on thread or tile bits become per-thread phases
    // that cost one multiply of every register per group that has any, so
    // gathering them into fewer groups saves those multiplies.
    if (!strict && gps.size() > 1 && defer_diag()) {
        const int G = (int)gps.size();
        std::vector<uint64_t> in_perm(G, 0), out_perm(G, 0);  // local bits the load / store maps touch
        for (int c = 0; c < G; ++c) {
            const GroupPlan &g = gps[c];
            uint64_t ti = g.qb, to = g.mb | g.permq;
            for (int j = 0; j < fm; ++j) {
                if (g.qcol[j] != (1 << j)) ti |= uint64_t(g.qcol[j] ^ (1 << j)) | (uint64_t(1) << j);
                if (g.mcol[j] != (1 << j)) to |= uint64_t(g.mcol[j] ^ (1 << j)) | (uint64_t(1) << j);
            }
            in_perm[c] = ti;
            out_perm[c] = to;
        }
        for (int c = 0; c + 1 < G; ++c) {
            std::vector<int> keep;
            const std::vector<int> gates = gps[c].gates;
            for (size_t k = 0; k < gates.size(); ++k) {
                const int q = gates[k];
                const GateMeta &m = meta[q];
                if (!m.diag) {
                    keep.push_back(q);
                    continue;
                }
                const uint64_t bits = gbits(m);
                bool later_conflict = false;  // a non-diagonal gate after it in this group
                for (size_t k2 = k + 1; k2 < gates.size() && !later_conflict; ++k2)
                    later_conflict = !meta[gates[k2]].diag && meta[gates[k2]].tl >= 0 &&
                                     ((bits >> meta[gates[k2]].tl) & 1);
                int dest = c;
                if (!later_conflict && !(out_perm[c] & bits)) {
                    for (int d = c + 1; d < G; ++d) {
                        if (in_perm[d] & bits) break;
                        dest = d;
                        bool blocked = (out_perm[d] & bits) != 0;
                        for (int q2 : gps[d].gates)  // (controls are diagonal: they commute)
                            if (!meta[q2].diag && meta[q2].tl >= 0 && ((bits >> meta[q2].tl) & 1)) blocked = true;
                        if (blocked) break;  // it goes first in d, before the conflict
                    }
                }
                if (dest == c)
                    keep.push_back(q);
                else
                    gps[dest].gates.insert(gps[dest].gates.begin(), q);
            }
            gps[c].gates = keep;
        }
    }
    if (gps.empty()) new_group();  // a pure layout pass (no gates)
    if (remap) {  // the last group stores through sigma o P
        GroupPlan &gl = gps.back();
        auto sg = [&](int x) {
            int y = 0;
            for (int b = 0; b < fm; ++b)
                if ((x >> b) & 1) y |= 1 << sig[b];
            return y;
        };
        for (int j = 0; j < fm; ++j) gl.mcol[j] = sg(gl.mcol[j]);
        gl.mb = sg(gl.mb);
    }
    // The last group stores straight to HBM; its rows stay whole 128 B lines
    // only if three non-slot local bits map (invertibly) onto local bits 0-2.
    // When its gate targets occupy them, a gate-free group is appended to
    // carry the store map: one more shared-memory transition (conflict-free)
    // costs less than uncoalesced HBM stores.
    auto low_cands = [&](const GroupPlan &g, std::vector<int> &out) {
        out.clear();
        for (int j = 0; j < fm; ++j)
            if (g.mcol[j] && !(g.mcol[j] >> 3) &&
                std::find(g.slots.begin(), g.slots.end(), j) == g.slots.end())
                out.push_back(j);
        for (size_t a = 0; a < out.size(); ++a)
            for (size_t b = a + 1; b < out.size(); ++b)
                for (size_t c = b + 1; c < out.size(); ++c) {
                    const int x = g.mcol[out[a]], y = g.mcol[out[b]], z = g.mcol[out[c]];
                    if (x != y && x != z && y != z && (x ^ y) != z) return true;
                }
        return false;
    };
    {
        std::vector<int> cands;
        if (!strict && !no_direct() && !gps.back().gates.empty() && !low_cands(gps.back(), cands)) {
            GroupPlan &gl = gps.back();
            int mcol[FMMAX], mb = gl.mb;
            for (int j = 0; j < fm; ++j) mcol[j] = gl.mcol[j], gl.mcol[j] = 1 << j;
            gl.mb = 0;
            GroupPlan *g2 = new_group();
            for (int j = 0; j < fm; ++j) g2->mcol[j] = mcol[j];
            g2->mb = mb;
        }
    }
    if ((int)gps.size() > FMAXGRP) return false;
    if (getenv("SVB_PLAN_DEBUG") && atoi(getenv("SVB_PLAN_DEBUG")) >= 2) {
        int nperm = 0;
        for (const GateMeta &m : meta) nperm += m.perm;
        fprintf(stderr, "pass: %d gates (%d X/CNOT), %zu groups:", ng, nperm, gps.size());
        for (const GroupPlan &g : gps) {
            fprintf(stderr, " [%zu gates, slots", g.gates.size());
            for (int s : g.slots) fprintf(stderr, " %d", s);
            fprintf(stderr, "%s]", g.permq ? ", perm" : "");
        }
        fprintf(stderr, "\n");
    }
    P.ngroups = (int)gps.size();
    int k0 = 0;
    for (int gi = 0; gi < P.ngroups; ++gi) {
        const GroupPlan &gp = gps[gi];
        int slots[FSMAX];
        int ns = 0;
        for (int s : gp.slots) slots[ns++] = s;
        // fill the free slots from the top, keeping off the local bits a
        // coalesced direct access needs as lanes (first group: bits 0-2; last
        // group: the bits its store map sends to 0-2)
        auto lane_bit = [&](int b) {
            if (gi == 0 && b < 3) return true;
            return gi == (int)gps.size() - 1 && gp.mcol[b] && !(gp.mcol[b] >> 3);
        };
        for (int pass2 = 0; pass2 < 2; ++pass2)
            for (int b = fm - 1; ns < fs && b >= 0; --b) {
                bool used = false;
                for (int i = 0; i < ns; ++i) used |= slots[i] == b;
                if (!used && (pass2 == 1 || !lane_bit(b))) slots[ns++] = b;
            }
        std::sort(slots, slots + fs);
        FGroup &G = P.groups[gi];
        for (int i = 0; i < fs; ++i) G.pos[i] = (int8_t)slots[i];
        G.first = (int16_t)k0;
        G.count = (int16_t)gp.gates.size();
        G.mb = (int16_t)gp.mb;
        G.perm = (int16_t)(gp.mb != 0 || gp.qb != 0);
        for (int j = 0; j < fm; ++j) {
            G.mcol[j] = (int16_t)gp.mcol[j];
            G.qcol[j] = (int16_t)gp.qcol[j];
            if (gp.mcol[j] != (1 << j) || gp.qcol[j] != (1 << j)) G.perm = 1;
        }
        G.qb = (int16_t)gp.qb;
        // can this group reach HBM directly (see direct_first / direct_last
        // below)?  Then its HBM side needs no bank-friendly lanes, and its
        // lanes 0-2 must stay on local bits 0-2.
        // Lanes 0-7 of a direct HBM access cover one 128 B line iff lanes 0-2
        // sit on three non-slot local bits that the group's map sends
        // (invertibly) into local bits 0-2, i.e. physical bits 0-2.
        bool is_slot_l[FMMAX] = {};
        for (int k = 0; k < fs; ++k) is_slot_l[slots[k]] = true;
        auto coal = [&](const int16_t *col, int *out) {
            if (no_direct()) return false;
            std::vector<int> cand;
            for (int j = 0; j < fm; ++j)
                if (!is_slot_l[j] && col[j] != 0 && (col[j] >> 3) == 0) cand.push_back(j);
            for (size_t a = 0; a < cand.size(); ++a)
                for (size_t b = a + 1; b < cand.size(); ++b)
                    for (size_t c = b + 1; c < cand.size(); ++c) {
                        const int x = col[cand[a]], y = col[cand[b]], z = col[cand[c]];
                        if (x != y && x != z && y != z && (x ^ y) != z) {
                            out[0] = cand[a], out[1] = cand[b], out[2] = cand[c];
                            return true;
                        }
                    }
            return false;
        };
        int pf[3], pl[3];
        const bool cf = gi == 0 && coal(G.qcol, pf);
        const bool cl = gi == P.ngroups - 1 && coal(G.mcol, pl);
        const int *pref = cl ? pl : (cf ? pf : nullptr);
        const bool same = cf && cl && pf[0] == pl[0] && pf[1] == pl[1] && pf[2] == pl[2];
        const bool can_df = cf && (!cl || same), can_dl = cl;
        // (an uncoalesced first group still reads shared memory when a JIT
        // pass prefetches tiles, so only coalesced direct sides skip the
        // bank-conflict search)
        // Only the shared-memory sides that use the fixed swizzle constrain
        // the lanes here -- group 0's loads (tiles filled by cp.async) and an
        // indirect last store; every transition between two groups gets its
        // own swizzle below.
        (void)can_df;
        (void)can_dl;
        thread_map(fm, fs, slots, G.tmap, G.qcol, G.mcol, gi == 0, gi == P.ngroups - 1 && !direct_any(), pref);
        auto slot_of = [&](int l) {
            for (int i = 0; i < fs; ++i)
                if (slots[i] == l) return i;
            return -1;
        };
        auto tbit_of = [&](int l) {  // local bit -> thread-index bit
            for (int j = 0; j < tbits; ++j)
                if (G.tmap[j] == l) return j;
            return -1;
        };
        for (size_t gk = 0; gk < gp.gates.size(); ++gk) {
            const GateMeta &m = meta[gp.gates[gk]];
            FGate &fg = P.gates[k0 + gk];
            for (int i = 0; i < 4; ++i) fg.m[i] = m.g.m[i];
            fg.u = 0;
            fg.tl = -1;
            int cs = m.cl >= 0 ? slot_of(m.cl) : -1;
            fg.cl = (int8_t)(m.cl >= 0 && cs < 0 ? tbit_of(m.cl) : -1);
            if (m.ct >= 0) fg.cl = (int8_t)(FTILEBIT + m.ct);  // control outside the tile
            fg.cmask = cs >= 0 ? slot_pattern(cs, fs) : 0xffffffffu;
            if (m.diag) {
                int ts = slot_of(m.tl);
                int tpos = ts >= 0 ? ts : FTPOS_THREAD;
                fg.tl = (int8_t)(ts >= 0 ? -1 : (m.tt >= 0 ? FTILEBIT + m.tt : tbit_of(m.tl)));
                int var = FD_GENERAL;
                if (m.g.d0_one) {
                    const int uc = unit_code(m.g.m[3]);
                    if (uc == 2)
                        var = FD_Z;
                    else if (kPermOps && uc == 1)
                        var = FD_S;
                    else if (kPermOps && uc == 3)
                        var = FD_SDG;
                    else
                        var = FD_D1;
                }
                if (kCompact && cs >= 0 && var == FD_Z) var = FD_D1;  // exact: cmul by (-1, 0)
                fg.op = (uint8_t)(FOP_DIAG + (var * (FSMAX + 1) + tpos) * 2 + (cs >= 0 ? 1 : 0));
            } else {
                int ts = slot_of(m.tl);
                int kind;
                switch (m.g.kind) {
                    case K_REAL: kind = FK_REAL; break;
                    case K_ANTI: kind = FK_ANTI; break;
                    case K_RX: kind = FK_RX; break;
                    default: kind = FK_GENERAL; break;
                }
                if (kPermOps && m.g.kind == K_ANTI) {
                    int u12 = unit_code(m.g.m[1]), u21 = unit_code(m.g.m[2]);
                    if (u12 == 0 && u21 == 0) {
                        kind = FK_X;
                    } else if (u12 == 3 && u21 == 1) {
                        kind = FK_Y;
                    } else if (u12 >= 0 && u21 >= 0) {
                        kind = FK_UANTI;
                        fg.u = (uint8_t)(u12 | (u21 << 2));
                    }
                }
                // pair loops visit lo registers (slot bit clear) whose control holds
                fg.cmask = fg.cmask & ~slot_pattern(ts, fs);
                if (kCompact && cs >= 0) kind = FK_GENERAL;  // general formula = reference's, exact
                fg.op = (uint8_t)((kind * FSMAX + ts) * 2 + (cs >= 0 ? 1 : 0));
            }
        }
        k0 += (int)gp.gates.size();
    }
    P.ngates = k0;

    // Shared-memory swizzle per transition.  A swizzle adds to a local index's
    // 16 B chunk number (bits 0-2) an XOR-linear function H of its higher
    // bits; any H is invertible.  The fill (cp.async) and the final copy use
    // the fixed fold3 one (H[j] = 1 << j % 3); between groups g and g+1 the
    // buffer is rewritten anyway, so H is searched such that g's STS.128 and
    // g+1's LDS.128 phases both hit 8 distinct bank groups.
    {
        const int G = P.ngroups;
        std::vector<std::array<int, FMMAX>> H(G + 1);  // H[t]: transition into group t (t = G: final copy)
        std::array<int, FMMAX> fold{};
        for (int j = 3; j < fm; ++j) fold[j] = 1 << (j % 3);
        auto bank = [&](int v, const std::array<int, FMMAX> &h) {
            int c = v & 7;
            for (int j = 3; j < fm; ++j)
                if ((v >> j) & 1) c ^= h[j];
            return c;
        };
        auto ways3 = [&](int a, int b, int c) {  // wavefronts of the 8-lane phase spanned by banks a, b, c
            int seen[8] = {0}, w = 0;
            for (int l = 0; l < 8; ++l) w = std::max(w, ++seen[((l & 1) ? a : 0) ^ ((l & 2) ? b : 0) ^ ((l & 4) ? c : 0)]);
            return w;
        };
        H[0] = fold;
        H[G] = fold;
        uint32_t rng = 0x9e3779b9u;
        for (int t = 1; t < G; ++t) {
            const FGroup &A = P.groups[t - 1], &B = P.groups[t];
            auto cost = [&](const std::array<int, FMMAX> &h) {
                return ways3(bank(A.mcol[A.tmap[0]], h), bank(A.mcol[A.tmap[1]], h), bank(A.mcol[A.tmap[2]], h)) +
                       ways3(bank(B.qcol[B.tmap[0]], h), bank(B.qcol[B.tmap[1]], h), bank(B.qcol[B.tmap[2]], h));
            };
            std::array<int, FMMAX> best = fold;
            int bc = cost(fold);
            for (int tries = 0; tries < 400 && bc > 2; ++tries) {
                std::array<int, FMMAX> h{};
                for (int j = 3; j < fm; ++j) {
                    rng = rng * 1664525u + 1013904223u;
                    h[j] = (rng >> 29) & 7;
                }
                const int c = cost(h);
                if (c < bc) {
                    bc = c;
                    best = h;
                }
            }
            H[t] = best;
        }
        auto off = [&](int v, const std::array<int, FMMAX> &h) {
            return (uint32_t)(16 * ((v & ~7) | bank(v, h)));
        };
        for (int gi = 0; gi < G; ++gi) {
            FGroup &Gr = P.groups[gi];
            const auto &hin = H[gi], &hout = H[gi + 1];
            for (int j = 0; j < tbits; ++j) {
                Gr.ld_t[j] = off(Gr.qcol[Gr.tmap[j]], hin);
                Gr.st_t[j] = off(Gr.mcol[Gr.tmap[j]], hout);
            }
            for (int k = 0; k < fs; ++k) {
                Gr.ld_s[k] = off(Gr.qcol[Gr.pos[k]], hin);
                Gr.st_s[k] = off(Gr.mcol[Gr.pos[k]], hout);
            }
            Gr.ld_b = off(Gr.qb, hin);
            Gr.st_b = off(Gr.mb, hout);
        }
    }

    // direct HBM access for the first / last group when the coalescing
    // condition holds: no slot on local bits 0-2, thread bits 0-2 = local bits
    // 0-2, and (last group) a store map that leaves bits 0-2 alone
    auto gidx = [&](int l) {
        int64_t g = 0;
        for (int b = 0; b < fm; ++b)
            if ((l >> b) & 1) g |= int64_t(1) << glob_of[b];
        return g;
    };
    // lanes 0-2 (local bits tmap[0..2]) map into local bits 0-2, invertibly
    auto coalesced = [&](const FGroup &G, const int16_t *col) {
        const int x = col[G.tmap[0]], y = col[G.tmap[1]], z = col[G.tmap[2]];
        if ((x | y | z) >> 3) return false;
        return x && y && z && x != y && x != z && y != z && (x ^ y) != z;
    };
    const FGroup &G0 = P.groups[0];
    P.direct_first = (coalesced(G0, G0.qcol) && !no_direct()) || direct_any();
    P.gl_b = gidx(G0.qb);
    for (int j = 0; j < tbits; ++j) P.gl_t[j] = gidx(G0.qcol[G0.tmap[j]]);
    for (int k = 0; k < fs; ++k) P.gl_s[k] = gidx(G0.qcol[G0.pos[k]]);
    const FGroup &GL = P.groups[P.ngroups - 1];
    P.direct_last = (coalesced(GL, GL.mcol) && !no_direct()) || direct_any();
    P.gs_b = gidx(GL.mb);
    for (int j = 0; j < tbits; ++j) P.gs_t[j] = gidx(GL.mcol[GL.tmap[j]]);
    for (int k = 0; k < fs; ++k) P.gs_s[k] = gidx(GL.mcol[GL.pos[k]]);
    return true;
}

static size_t fused_smem() { return kNBuf * FTILE * sizeof(double2) + FMAXROWS * sizeof(int64_t); }

static int fused_grid(int64_t ntiles) {
    static int sms = [] {
        int d = 0, v = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        return v;
    }();
    return (int)std::min<int64_t>(ntiles, int64_t(sms) * FCTAS_PER_SM);
}

static bool fuse_enabled(int n, unsigned flags) { return (flags & SVB_RUN_FUSE) && n >= FM + 2; }

int jit_compile_only(const std::vector<FPass> &passes, int variant, std::string &err);
int jit_variant(bool fma);
bool jit_available();

// Tile qubits of a plan: the interpreter's FM, or -- for runtime-specialised
// passes -- 12 while the state still has >= 2^12 tiles (every SM busy):
// bigger tiles hold more qubits, so fewer HBM passes per circuit.  configs[1]
// measured: fm 11 239 passes x 0.416 ms = 77.2k gate apps/s, fm 12 203 x
// 0.467 ms = 81.0k, fm 13 174 x 0.574 ms = 77.0k (one 512-thread CTA per SM
// hides latency worse).  SVB_JIT_FM overrides (11..FMMAX).
static int plan_fm(int n, unsigned flags) {
    if (!(flags & SVB_RUN_JIT) || !jit_available()) return FM;
    const char *e = getenv("SVB_JIT_FM");
    const int fm = e ? atoi(e) : std::min(12, n - 12);
    return std::max(FM, std::min(FMMAX, fm));
}

// Slot bits per thread of a plan: FSLOTS for the interpreter; specialised
// passes hold 32 amplitudes per thread (5 slots, 255 registers, 2 CTAs of
// 128 threads per SM at fm 12): fewer register groups -- each a full
// shared-memory transposition of the tile -- per pass.  SVB_JIT_FS overrides.
static int plan_fs(unsigned flags) {
    if (!(flags & SVB_RUN_JIT) || !jit_available()) return FSLOTS;
    const char *e = getenv("SVB_JIT_FS");
    const int fs = e ? atoi(e) : 5;
    return std::max(4, std::min(FSMAX, fs));
}

// Ops with Z-type qubits outside the tile (need_mask): specialised passes
// only -- the interpreter has no tile-uniform predicates.  SVB_FUSE_OUTSIDE=0
// turns it off (measurement).
static bool plan_outside(unsigned flags) {
    if (!(flags & SVB_RUN_JIT) || (flags & SVB_RUN_STRICT_ORDER) || !jit_available()) return false;
    const char *e = getenv("SVB_FUSE_OUTSIDE");
    return !e || atoi(e) != 0;
}

struct PlanStep {
    int op;      // >= 0: run `mapped` (ops[op] on physical qubits) with the single-gate kernels
    svb_op mapped;
    // -1: next fused pass
};

// shared-memory wavefronts of one 8-lane LDS/STS.128 phase (1 = conflict-free)
static int phase_ways(const uint32_t *t) {
    int seen[8] = {0}, w = 0;
    for (int l = 0; l < 8; ++l) {
        unsigned a = 0;
        for (int j = 0; j < 3; ++j)
            if ((l >> j) & 1) a ^= t[j];
        w = std::max(w, ++seen[(a >> 4) & 7]);
    }
    return w;
}

// Plan an op list and lower it to steps + pass descriptors, tracking the
// qubit layout: non-strict plans let each pass move three qubits of the next
// pass's set to physical bits 0-2 (so no qubit is pinned into every tile:
// configs[1] 203 -> 170 passes at fm 12), the others of its set go home
// when they can, and gate-free layout passes at the end restore the
// identity layout the caller expects.
static void lower_plan(int n, const svb_op *ops, int nops, bool strict, bool regperm, int fm, int fs,
                       bool outside, std::vector<PlanStep> &steps, std::vector<FPass> &passes,
                       int kind = planner_kind()) {
    outside = outside && !strict && kind == 3;
    const auto t_plan0 = std::chrono::steady_clock::now();
    const std::vector<PlanPass> plans = plan(n, ops, nops, strict, fm, outside, kind);
    if (getenv("SVB_PLAN_DEBUG"))
        fprintf(stderr, "plan: op grouping %.3f s\n",
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t_plan0).count());
    const int nlow = flow_bits();
    const bool rotate = !strict && rotate_low() && kind == 3;
    std::vector<int8_t> phys(64), nxt(64);
    for (int q = 0; q < 64; ++q) phys[q] = (int8_t)q;
    auto single = [&](int oi) {
        PlanStep st;
        st.op = oi;
        st.mapped = ops[oi];
        st.mapped.target = phys[ops[oi].target];
        if (ops[oi].kind == 1) st.mapped.control = phys[ops[oi].control];
        steps.push_back(st);
    };
    auto fused = [&](const PlanPass &pp, const int8_t *next) {
        FPass P;
        if (!build_pass(n, ops, pp, P, strict, regperm, fm, phys.data(), next, fs)) return false;
        PlanStep st;
        st.op = -1;
        memset(&st.mapped, 0, sizeof st.mapped);
        steps.push_back(st);
        passes.push_back(P);
        if (next) phys.assign(next, next + 64);
        return true;
    };
    for (size_t k = 0; k < plans.size(); ++k) {
        const PlanPass &pp = plans[k];
        // (with a rotating layout even a one-op pass runs as a tile pass: it
        // is the pass that brings the next pass's qubits to bits 0-2)
        if (pp.ops.size() <= 1 && !rotate) {
            for (int oi : pp.ops) single(oi);
            continue;
        }
        const int8_t *next = nullptr;
        if (rotate) {
            // new physical bits 0..nlow-1: nlow qubits of this set that the next
            // pass also tiles (the planner guarantees >= nlow), those already
            // low first; among the choices, the first whose last-group store
            // stays coalesced (its lanes need the new low qubits off the slots)
            const uint64_t want = k + 1 < plans.size() ? (pp.S & plans[k + 1].S) : (pp.S & ((1ull << nlow) - 1));
            std::vector<int> pool;
            for (int pass2 = 0; pass2 < 2; ++pass2)
                for (int q = 0; q < n; ++q)
                    if (((want >> q) & 1) && ((phys[q] < nlow) == (pass2 == 0))) pool.push_back(q);
            for (int q = 0; q < n && (int)pool.size() < nlow; ++q)  // (last pass: any current low qubit)
                if (((pp.S >> q) & 1) && phys[q] < nlow && std::find(pool.begin(), pool.end(), q) == pool.end())
                    pool.push_back(q);
            std::vector<std::vector<int>> choices;
            const int np = (int)pool.size();
            for (int a = 0; a < np && choices.size() < 24; ++a)
                for (int b = a + 1; b < np && choices.size() < 24; ++b)
                    for (int c = b + 1; c < np && choices.size() < 24; ++c)
                        if (nlow == 3) choices.push_back({pool[a], pool[b], pool[c]});
            if (choices.empty()) choices.push_back(std::vector<int>(pool.begin(), pool.begin() + std::min(np, nlow)));
            // every choice is lowered (build_pass: register groups, swizzle
            // search) independently on up to 16 host threads; the lowest
            // score wins, the first in choice order on ties
            const size_t nc = choices.size();
            std::vector<FPass> cand(nc);
            std::vector<std::vector<int8_t>> cand_next(nc);
            std::vector<int> cand_score(nc, 1 << 20);
            auto lower_one = [&](size_t ci) {
            const std::vector<int> &lowq = choices[ci];
            std::vector<int8_t> nx = phys;
            uint64_t T = 0;  // the tile's physical bits
            for (int q = 0; q < n; ++q)
                if ((pp.S >> q) & 1) T |= uint64_t(1) << phys[q];
            uint64_t taken = 0;
            std::vector<int> rest;
            for (int q : lowq)  // already-low ones keep their bit
                if (phys[q] < nlow) taken |= uint64_t(1) << phys[q];
            for (int q : lowq)
                if (phys[q] >= nlow) {
                    int b = 0;
                    while ((taken >> b) & 1) ++b;
                    nx[q] = (int8_t)b;
                    taken |= uint64_t(1) << b;
                }
            for (int q = 0; q < n; ++q) {
                if (!((pp.S >> q) & 1) || std::find(lowq.begin(), lowq.end(), q) != lowq.end()) continue;
                if (q >= nlow && ((T >> q) & 1) && !((taken >> q) & 1)) {
                    nx[q] = (int8_t)q;  // home
                    taken |= uint64_t(1) << q;
                } else {
                    rest.push_back(q);
                }
            }
            for (int q : rest) {
                int b = 0;
                while (!((T >> b) & 1) || ((taken >> b) & 1)) ++b;
                nx[q] = (int8_t)b;
                taken |= uint64_t(1) << b;
            }
            FPass &P = cand[ci];
            if (!build_pass(n, ops, pp, P, strict, regperm, fm, phys.data(), nx.data(), fs)) return;
            // score: uncoalesced last-group HBM store (2) + shared-memory
            // conflicts of the last group's loads and the groups' stores
            const FGroup &GL = P.groups[P.ngroups - 1];
            const int x = GL.mcol[GL.tmap[0]], y = GL.mcol[GL.tmap[1]], z = GL.mcol[GL.tmap[2]];
            const bool coal = !((x | y | z) >> 3) && (x | y | z) == 7 && x != y && x != z && y != z && (x ^ y) != z;
            // (a gate-free last group was appended when the store could not
            // be coalesced otherwise: fewer groups first)
            int score = 4 * P.ngroups + (coal ? 0 : 2);
            score += phase_ways(GL.ld_t) - 1;
            for (int gi = 0; gi + 1 < P.ngroups; ++gi) score += phase_ways(P.groups[gi].st_t) - 1;
            cand_score[ci] = score;
            cand_next[ci] = std::move(nx);
            };
            const unsigned nthr = std::min<unsigned>((unsigned)nc,
                                                     std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
            if (nthr > 1) {
                std::atomic<size_t> nextc{0};
                std::vector<std::thread> pool;
                for (unsigned t = 1; t < nthr; ++t)
                    pool.emplace_back([&] {
                        for (size_t c; (c = nextc++) < nc;) lower_one(c);
                    });
                for (size_t c; (c = nextc++) < nc;) lower_one(c);
                for (auto &t : pool) t.join();
            } else {
                for (size_t c = 0; c < nc; ++c) lower_one(c);
            }
            bool built = false;
            size_t bi = 0;
            for (size_t ci = 0; ci < nc; ++ci)
                if (cand_score[ci] < (built ? cand_score[bi] : (1 << 20))) {
                    bi = ci;
                    built = true;
                }
            FPass best;
            std::vector<int8_t> best_next;
            if (built) {
                best = cand[bi];
                best_next = cand_next[bi];
            }
            if (built) {
                PlanStep st;
                st.op = -1;
                memset(&st.mapped, 0, sizeof st.mapped);
                steps.push_back(st);
                passes.push_back(best);
                phys = best_next;
            } else {
                for (int oi : pp.ops) single(oi);
            }
            continue;
        }
        if (!fused(pp, next))
            for (int oi : pp.ops) single(oi);
    }
    // restore the identity layout with gate-free passes
    for (int guard = 0; guard < 64; ++guard) {
        std::vector<int> inv(n);
        uint64_t disp = 0;
        for (int q = 0; q < n; ++q) {
            inv[phys[q]] = q;
            if (phys[q] != q) disp |= uint64_t(1) << phys[q];
        }
        if (!disp) break;
        uint64_t T = (uint64_t(1) << nlow) - 1;
        // whole cycles while they fit, then a segment of the next one
        for (int p0 = 0; p0 < n && popc(T) < fm; ++p0) {
            if (!((disp >> p0) & 1) || ((T >> p0) & 1 && p0 >= nlow)) continue;
            for (int p = p0; popc(T) < fm; p = inv[p]) {
                T |= uint64_t(1) << p;
                if (inv[p] == p0) break;
            }
        }
        for (int b = n - 1; b >= 0 && popc(T) < fm; --b) T |= uint64_t(1) << b;
        PlanPass pp;
        for (int b = 0; b < n; ++b)
            if ((T >> b) & 1) pp.S |= uint64_t(1) << inv[b];
        nxt = phys;
        uint64_t taken = 0;
        std::vector<int> rest;
        for (int b = 0; b < n; ++b) {
            if (!((T >> b) & 1)) continue;
            const int q = inv[b];
            if ((T >> q) & 1) {
                nxt[q] = (int8_t)q;
                taken |= uint64_t(1) << q;
            } else {
                rest.push_back(q);
            }
        }
        for (int q : rest) {
            int b = 0;
            while (!((T >> b) & 1) || ((taken >> b) & 1)) ++b;
            nxt[q] = (int8_t)b;
            taken |= uint64_t(1) << b;
        }
        if (!fused(pp, nxt.data())) break;  // cannot happen: a gate-free pass always builds
    }
}

// host-only: plan, lower and NVRTC-compile every fused pass (no device work)
// ---------------------------------------------------------------------------
// Trailing SWAP network in one HBM pass.
//
// A circuit that ends in SWAPs written as CNOT triples (the reference's form:
// the QFT's final qubit reversal, core.py / workloads.qft_circuit) permutes
// the bits of every amplitude index.  Through fused passes that costs one
// pass per ~4-6 swaps (both qubits of a swap must share a 12-qubit tile that
// also holds physical bits 0-2): QFT-30 spent 3 of its 7 passes moving data
// for the reversal.  When the swaps are pairwise disjoint and each of the K
// lowest qubits is swapped with a qubit >= K, the whole network is done in
// place in ONE pass: split the index into the low block A (bits 0..K-1), its
// partners B and the rest R; the network maps tile r (all 2^K x 2^K
// combinations of A and B bits) to the transposed tile at sigma_R(r).  A CTA
// loads tile r and its partner tile into shared memory as 2^K rows of 2^K
// contiguous amplitudes (512 B at K = 5) and stores each transposed into the
// other's place.  Pure data movement: bit-identical to applying the CNOTs.
struct SwapNet {
    int n, nrest, npairs;
    int8_t hi[8];         // partner (>= K) of low qubit i
    int8_t rest[64];      // qubits outside A and B, ascending = bit j of the tile index
    int rev;              // the swaps inside R reverse the tile index: partner tile = bit reversal
    int nruns;            // ... as runs of consecutive qubits: tile bits [off, off+len) -> qubits [pos, pos+len)
    int8_t run_off[16], run_len[16], run_pos[16];
    int8_t pu[32], pv[32];  // swaps inside R, as tile-index bit positions
};
constexpr int SWAPNET_K = 5;

__global__ void __launch_bounds__(256) k_swap_bits(double2 *__restrict__ a, SwapNet w) {
    constexpr int K = SWAPNET_K, T = 1 << K;
    __shared__ double2 s1[T][T + 1], s2[T][T + 1];  // [B value][A value], padded: transposed reads hit 8 bank groups
    const int64_t ntiles = int64_t(1) << w.nrest;
    // Tiles are visited in an order whose fastest bits are the tile index's
    // lowest J and highest J bits: for a reversal-like network the partners of
    // the tiles in flight then lie in the same small set of 2 MB pages as the
    // tiles themselves (in plain order the partners of consecutive tiles are
    // spread over the whole state: 3.5 TB/s on QFT-30, TLB-bound).
    int64_t yo[(T * T) / 256];  // row offsets of this thread's elements: the B bits of their row number
#pragma unroll
    for (int r = 0; r < (T * T) / 256; ++r) {
        const int y = (threadIdx.x + r * 256) >> K;
        int64_t o = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) o |= int64_t((y >> i) & 1) << w.hi[i];
        yo[r] = o;
    }
    const int J = w.nrest >= 10 ? 5 : w.nrest / 2;
    const int64_t jm = (int64_t(1) << J) - 1;
    for (int64_t u = blockIdx.x; u < ntiles; u += gridDim.x) {
        const int64_t t = (u & jm) | (((u >> J) & jm) << (w.nrest - J)) | ((u >> (2 * J)) << J);
        int64_t tp = t;
        if (w.rev) {
            tp = (int64_t)(__brevll((unsigned long long)t) >> (64 - w.nrest));
        } else {
            for (int j = 0; j < w.npairs; ++j)
                if (((t >> w.pu[j]) ^ (t >> w.pv[j])) & 1) tp ^= (int64_t(1) << w.pu[j]) | (int64_t(1) << w.pv[j]);
        }
        if (tp < t) continue;  // a pair of tiles is exchanged at its lower index
        int64_t base = 0, basep = 0;
        for (int j = 0; j < w.nruns; ++j) {
            const int64_t m = (int64_t(1) << w.run_len[j]) - 1;
            base |= ((t >> w.run_off[j]) & m) << w.run_pos[j];
            basep |= ((tp >> w.run_off[j]) & m) << w.run_pos[j];
        }
#pragma unroll
        for (int r = 0; r < (T * T) / 256; ++r) {
            const int e = threadIdx.x + r * 256, x = e & (T - 1), y = e >> K;
            s1[y][x] = a[base + yo[r] + x];
            if (tp != t) s2[y][x] = a[basep + yo[r] + x];
        }
        __syncthreads();
        // the amplitude the network puts at (A = x, B = y) of tile tp comes from (A = y, B = x) of tile t
#pragma unroll
        for (int r = 0; r < (T * T) / 256; ++r) {
            const int e = threadIdx.x + r * 256, x = e & (T - 1), y = e >> K;
            a[basep + yo[r] + x] = s1[x][y];
            if (tp != t) a[base + yo[r] + x] = s2[x][y];
        }
        __syncthreads();
    }
}

static bool swapnet_on() {
    static const bool on = [] {
        const char *e = getenv("SVB_FUSE_SWAPNET");
        return !e || atoi(e) != 0;
    }();
    return on;
}

// Length (in ops, a multiple of 3) of the trailing SWAP network that
// k_swap_bits applies, 0 if the ops do not end in one that qualifies.
int swap_suffix(int n, const svb_op *ops, int nops, SwapNet *out) {
    constexpr int K = SWAPNET_K;
    if (!swapnet_on() || n < 2 * K + 2 || n > 62) return 0;
    auto is_cx = [&](const svb_op &o, int c, int t) {
        static const double X[8] = {0, 0, 1, 0, 1, 0, 0, 0};
        return o.kind == 1 && o.control == c && o.target == t && memcmp(o.q, X, sizeof X) == 0;
    };
    int sigma[64];
    for (int q = 0; q < n; ++q) sigma[q] = q;
    int i = nops, swaps = 0;
    while (i >= 3) {
        const svb_op &o = ops[i - 1];
        if (o.kind != 1) break;
        const int c = o.control, t = o.target;
        if (c == t || c < 0 || t < 0 || c >= n || t >= n) break;
        if (!is_cx(ops[i - 1], c, t) || !is_cx(ops[i - 2], t, c) || !is_cx(ops[i - 3], c, t)) break;
        if (sigma[c] != c || sigma[t] != t) break;  // not disjoint from the swaps taken so far
        sigma[c] = t;
        sigma[t] = c;
        i -= 3;
        ++swaps;
    }
    // worth a dedicated pass only for a network (a few swaps relabel for free inside fused passes)
    if (swaps < 3) return 0;
    for (int q = 0; q < K; ++q)
        if (sigma[q] < K) return 0;  // the low block must move out whole
    if (out) {
        SwapNet &w = *out;
        memset(&w, 0, sizeof w);
        w.n = n;
        bool in_b[64] = {false};
        for (int q = 0; q < K; ++q) {
            w.hi[q] = (int8_t)sigma[q];
            in_b[sigma[q]] = true;
        }
        int pos[64];
        for (int q = K; q < n; ++q)
            if (!in_b[q]) {
                pos[q] = w.nrest;
                w.rest[w.nrest++] = (int8_t)q;
            }
        for (int j = 0; j < w.nrest; ++j) {
            if (j > 0 && w.rest[j] == w.rest[j - 1] + 1) {
                ++w.run_len[w.nruns - 1];
                continue;
            }
            if (w.nruns >= 16) return 0;
            w.run_off[w.nruns] = (int8_t)j;
            w.run_len[w.nruns] = 1;
            w.run_pos[w.nruns] = w.rest[j];
            ++w.nruns;
        }
        for (int q = K; q < n; ++q)
            if (!in_b[q] && sigma[q] > q) {
                if (w.npairs >= 32) return 0;
                w.pu[w.npairs] = (int8_t)pos[q];
                w.pv[w.npairs] = (int8_t)pos[sigma[q]];
                ++w.npairs;
            }
        w.rev = w.nrest >= 2 && w.npairs == w.nrest / 2;
        for (int j = 0; j < w.npairs; ++j)
            if (w.pu[j] + w.pv[j] != w.nrest - 1) w.rev = 0;
    }
    return nops - i;
}

int jit_check(int n, const svb_op *ops, int nops, unsigned flags) {
    if (fuse_enabled(n, flags | SVB_RUN_FUSE)) nops -= swap_suffix(n, ops, nops, nullptr);  // (k_swap_bits runs the rest)
    const bool strict = flags & SVB_RUN_STRICT_ORDER;
    std::vector<FPass> passes;
    std::vector<PlanStep> steps;
    const int fm = plan_fm(n, flags | SVB_RUN_JIT);
    lower_plan(n, ops, nops, strict, reg_perm(flags | SVB_RUN_JIT), fm, plan_fs(flags | SVB_RUN_JIT),
               plan_outside(flags | SVB_RUN_JIT), steps, passes);
    std::string err;
    int r = jit_compile_only(passes, jit_variant((flags & SVB_RUN_FMA) && !strict), err);
    if (r < 0) set_error("jit compile failed: %.400s", err.c_str());
    return r;
}

int plan_passes(int n, const svb_op *ops, int nops, unsigned flags, int *groups) {
    if (groups) *groups = 0;
    if (!fuse_enabled(n, flags)) return nops;
    const int tail = swap_suffix(n, ops, nops, nullptr);  // one k_swap_bits pass
    if (tail) return plan_passes(n, ops, nops - tail, flags, groups) + 1;
    const bool strict = flags & SVB_RUN_STRICT_ORDER;
    const int fm = plan_fm(n, flags);
    std::vector<FPass> passes;
    std::vector<PlanStep> steps;
    lower_plan(n, ops, nops, strict, reg_perm(flags), fm, plan_fs(flags), plan_outside(flags), steps, passes);
    int df = 0, dl = 0, cf = 0, cl = 0;
    auto coal = [](const FGroup &G, const int16_t *col) {
        const int x = col[G.tmap[0]], y = col[G.tmap[1]], z = col[G.tmap[2]];
        return !((x | y | z) >> 3) && (x | y | z) == 7 && x != y && x != z && y != z && (x ^ y) != z;
    };
    const bool dbg3 = getenv("SVB_PLAN_DEBUG") && atoi(getenv("SVB_PLAN_DEBUG")) >= 3;
    auto ways = [](const uint32_t *t) {  // wavefronts per LDS/STS.128 phase of 8 lanes (1 = conflict-free)
        int seen[8] = {0}, w = 0;
        for (int l = 0; l < 8; ++l) {
            unsigned a = 0;
            for (int j = 0; j < 3; ++j)
                if ((l >> j) & 1) a ^= t[j];
            w = std::max(w, ++seen[(a >> 4) & 7]);
        }
        return w;
    };
    for (const FPass &P : passes) {
        if (groups) *groups += P.ngroups;
        df += P.direct_first;
        dl += P.direct_last;
        const bool c0 = coal(P.groups[0], P.groups[0].qcol), c1 = coal(P.groups[P.ngroups - 1], P.groups[P.ngroups - 1].mcol);
        cf += c0;
        cl += c1;
        if (dbg3) {
            // distinct non-diagonal targets: a lower bound of ceil(targets / fs) groups
            uint32_t tg = 0;
            for (int gi = 0; gi < P.ngroups; ++gi) {
                const FGroup &G = P.groups[gi];
                for (int q = G.first; q < G.first + G.count; ++q)
                    if (P.gates[q].op < FOP_DIAG) tg |= 1u << G.pos[(P.gates[q].op >> 1) % FSMAX];
            }
            fprintf(stderr, "pass: %d gates, %d groups, %d targets, coalesced %d %d | banks:", P.ngates, P.ngroups,
                    __builtin_popcount(tg), c0, c1);
            for (int gi = 0; gi < P.ngroups; ++gi) {
                const FGroup &G = P.groups[gi];
                // JIT passes with prefetch read group 0 from shared memory too
                const bool st_smem = !(gi == P.ngroups - 1 && P.direct_last);
                fprintf(stderr, " g%d ld %d st %d", gi, ways(G.ld_t), st_smem ? ways(G.st_t) : 0);
            }
            fprintf(stderr, "\n");
        }
    }
    if (getenv("SVB_PLAN_DEBUG"))
        fprintf(stderr,
                "plan: %zu steps (%zu fused passes), %d groups, direct first %d (coalesced %d), "
                "direct last %d (coalesced %d)\n",
                steps.size(), passes.size(), groups ? *groups : -1, df, cf, dl, cl);
    return (int)steps.size();
}

// ---------------------------------------------------------------------------
// compiled plans, cached: a circuit run repeatedly (bench steps, parameter
// sweeps) is planned and lowered to kernel descriptors once.

struct CompiledPlan {
    int n, fm, fs, kind;
    bool strict, regperm, outside;
    std::vector<svb_op> ops;  // exact key
    std::vector<PlanStep> steps;
    std::vector<FPass> passes;
    // runtime-specialised kernels per pass (jit.cu), built on first JIT use
    mutable std::mutex jit_mu;
    // per variant (exact / FMA / FMA + factors): 0 untried, 1 built, -1 failed
    mutable int jit_state[3] = {0, 0, 0};
    mutable std::vector<void *> jit_fns[3];
    mutable std::vector<std::shared_ptr<void>> jit_keep[3];  // the loaded modules (unloaded with the plan)
    // devices this plan's JIT kernels were launched on: before the modules are
    // released (and unloaded), those devices are drained, so no launch of a
    // module can still be queued when cudaLibraryUnload runs
    mutable std::atomic<uint64_t> jit_devices{0};
    ~CompiledPlan() {
        const uint64_t m = jit_devices.load();
        if (!m) return;
        int cur = 0;
        if (cudaGetDevice(&cur) != cudaSuccess) return;
        for (int d = 0; d < 64; ++d)
            if ((m >> d) & 1) {
                cudaSetDevice(d);
                cudaDeviceSynchronize();
            }
        cudaSetDevice(cur);
        cudaGetLastError();
    }
};

bool jit_build(const std::vector<FPass> &passes, int variant, std::vector<void *> &fns,
               std::vector<std::shared_ptr<void>> &keep);
void jit_async(std::function<void()> fn);
bool jit_launch(void *fn, const FPass &P, double2 *a, int64_t ntiles, cudaStream_t s);

static uint64_t fnv1a(const void *p, size_t len, uint64_t h) {
    const unsigned char *b = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < len; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

// descriptor bytes the plan cache keeps beyond its 4 most recent plans
// (SVB_PLAN_CACHE_MB, default 256; read per call)
static size_t plan_cache_bytes() {
    const char *e = getenv("SVB_PLAN_CACHE_MB");
    return (e ? size_t(atoll(e)) : size_t(256)) << 20;
}

static std::shared_ptr<const CompiledPlan> compiled_plan(int n, const svb_op *ops, int nops, bool strict,
                                                         bool regperm, int fm, int fs, bool outside,
                                                         int kind = planner_kind(), bool peek = false) {
    // (never destroyed: a background compile still running at process exit
    // may use them after static destruction began)
    static std::mutex &mu = *new std::mutex;
    static auto &cache = *new std::vector<std::pair<uint64_t, std::shared_ptr<const CompiledPlan>>>;  // MRU first
    uint64_t key = fnv1a(ops, sizeof(svb_op) * size_t(nops), 1469598103934665603ull);
    key = fnv1a(&n, sizeof n, key);
    key = fnv1a(&strict, sizeof strict, key);
    key = fnv1a(&regperm, sizeof regperm, key);
    key = fnv1a(&fm, sizeof fm, key);
    key = fnv1a(&fs, sizeof fs, key);
    key = fnv1a(&outside, sizeof outside, key);
    key = fnv1a(&kind, sizeof kind, key);
    {
        std::lock_guard<std::mutex> lk(mu);
        for (size_t i = 0; i < cache.size(); ++i) {
            const auto &c = cache[i].second;
            if (cache[i].first == key && c->n == n && c->fm == fm && c->fs == fs && c->outside == outside &&
                c->strict == strict && c->regperm == regperm && c->kind == kind && (int)c->ops.size() == nops &&
                std::memcmp(c->ops.data(), ops, sizeof(svb_op) * size_t(nops)) == 0) {
                auto hit = cache[i];
                cache.erase(cache.begin() + i);
                cache.insert(cache.begin(), hit);
                return hit.second;
            }
        }
    }
    if (peek) return nullptr;
    auto cp = std::make_shared<CompiledPlan>();
    cp->n = n;
    cp->fm = fm;
    cp->fs = fs;
    cp->kind = kind;
    cp->strict = strict;
    cp->regperm = regperm;
    cp->outside = outside;
    cp->ops.assign(ops, ops + nops);
    lower_plan(n, ops, nops, strict, regperm, fm, fs, outside, cp->steps, cp->passes, kind);
    // Bounded by descriptor bytes (~27 KiB per pass), not by count: the
    // multi-process engine runs one op segment per exchange interval, so a
    // circuit step may cycle through hundreds of small plans.
    std::lock_guard<std::mutex> lk(mu);
    cache.insert(cache.begin(), {key, cp});
    size_t bytes = 0, keep = 0;
    for (; keep < cache.size(); ++keep) {
        bytes += cache[keep].second->passes.size() * sizeof(FPass) + cache[keep].second->ops.size() * sizeof(svb_op);
        if (keep >= 4 && bytes > plan_cache_bytes()) break;
    }
    cache.resize(std::max<size_t>(keep, 1));
    return cp;
}

// SVB_RUN_JIT_ASYNC: plan + compile the specialised passes of an op list on
// a background thread (once per op list: in-flight keys are remembered).
// The plan lands in the plan cache with its kernels already built, so a later
// call finds it through compiled_plan(..., peek) with jit_state 1.
static bool start_async_jit(int n, const svb_op *ops, int nops, bool strict, bool regperm, int fm, int fs,
                            bool outside, int variant) {
    static std::mutex &mu = *new std::mutex;  // (never destroyed, as the plan cache)
    static std::vector<uint64_t> &inflight = *new std::vector<uint64_t>;
    uint64_t key = fnv1a(ops, sizeof(svb_op) * size_t(nops), 0x2545f4914f6cdd1dull);
    key = fnv1a(&n, sizeof n, key);
    key = fnv1a(&variant, sizeof variant, key);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (std::find(inflight.begin(), inflight.end(), key) != inflight.end()) return false;
        inflight.push_back(key);
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::vector<svb_op> copy(ops, ops + nops);
    jit_async([copy = std::move(copy), n, strict, regperm, fm, fs, outside, variant, dev, key] {
        cudaSetDevice(dev);
        std::shared_ptr<const CompiledPlan> cp =
            compiled_plan(n, copy.data(), (int)copy.size(), strict, regperm, fm, fs, outside);
        {
            std::lock_guard<std::mutex> lk2(cp->jit_mu);
            if (cp->jit_state[variant] == 0)
                cp->jit_state[variant] =
                    jit_build(cp->passes, variant, cp->jit_fns[variant], cp->jit_keep[variant]) ? 1 : -1;
        }
        std::lock_guard<std::mutex> lk(mu);
        inflight.erase(std::find(inflight.begin(), inflight.end(), key));
    });
    return true;
}

int run_ops_device(double2 *a, int64_t n_amps, const svb_op *ops, int nops, unsigned flags,
                   cudaStream_t s, int64_t *launches) {
    int n = 0;
    while ((int64_t(1) << n) < n_amps) ++n;
    auto single = [&](const svb_op &o) {
        prof_begin(s);
        LaunchInfo li = launch_gate(a, n_amps, make_gate(o.q), o.target, o.kind == 1 ? o.control : -1, s);
        prof_end(s, li);
        *launches += li.kernels;
    };
    if (!fuse_enabled(n, flags)) {
        for (int i = 0; i < nops; ++i) single(ops[i]);
        return SVB_OK;
    }
    SwapNet net;
    const int tail = swap_suffix(n, ops, nops, &net);
    if (tail) {
        // the ops before the network through the usual plan, then the network in one pass
        int r = nops > tail ? run_ops_device(a, n_amps, ops, nops - tail, flags, s, launches) : SVB_OK;
        if (r != SVB_OK) return r;
        static const int sms = [] {
            int d = 0, v = 148;
            cudaGetDevice(&d);
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
            return v;
        }();
        const int64_t ntiles = int64_t(1) << net.nrest;
        prof_begin(s);
        k_swap_bits<<<(unsigned)std::min<int64_t>(ntiles, int64_t(sms) * 6), 256, 0, s>>>(a, net);
        prof_end(s, LaunchInfo{1, PROF_SWAPNET, n_amps * 32});
        *launches += 1;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "k_swap_bits launch");
        return SVB_OK;
    }
    {  // the dynamic shared-memory opt-in is per device: set it for each device used
        static std::atomic<uint64_t> attr_set{0};
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
        if (!(attr_set.load() & bit)) {
            cudaFuncSetAttribute(k_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem());
            cudaFuncSetAttribute(k_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem());
            attr_set.fetch_or(bit);
        }
    }
    const bool strict = flags & SVB_RUN_STRICT_ORDER;
    const bool fma = (flags & SVB_RUN_FMA) && !strict;
    const int variant = jit_variant(fma);
    std::shared_ptr<const CompiledPlan> cp;
    if ((flags & SVB_RUN_JIT) && (flags & SVB_RUN_JIT_ASYNC) && jit_available()) {
        // use the specialised plan only once its kernels are built; until
        // then a quickly planned interpreter run (lookahead planner: ~0.07 s
        // for configs[1] instead of ~1 s) while a background thread plans and
        // compiles the specialised one
        cp = compiled_plan(n, ops, nops, strict, reg_perm(flags), plan_fm(n, flags), plan_fs(flags),
                           plan_outside(flags), planner_kind(), true);
        int state = 0;
        if (cp) {
            std::lock_guard<std::mutex> lk(cp->jit_mu);
            state = cp->jit_state[variant];
        }
        if (state != 1) {
            if (state == 0)
                start_async_jit(n, ops, nops, strict, reg_perm(flags), plan_fm(n, flags), plan_fs(flags),
                                plan_outside(flags), variant);
            cp = compiled_plan(n, ops, nops, strict, reg_perm(flags & ~SVB_RUN_JIT), FM, FSLOTS, false,
                               strict ? planner_kind() : 2);
            flags &= ~(SVB_RUN_JIT | SVB_RUN_JIT_ASYNC);
        }
    }
    if (!cp)
        cp = compiled_plan(n, ops, nops, strict, reg_perm(flags), plan_fm(n, flags), plan_fs(flags),
                           plan_outside(flags));
    size_t next_pass = 0;
    bool jit = (flags & SVB_RUN_JIT) && !cp->passes.empty();
    const std::vector<void *> *jit_fns = nullptr;
    if (jit) {
        std::lock_guard<std::mutex> lk(cp->jit_mu);
        int &state = cp->jit_state[variant];
        if (state == 0)
            state = jit_build(cp->passes, variant, cp->jit_fns[variant], cp->jit_keep[variant]) ? 1 : -1;
        if (state == 1) {
            jit_fns = &cp->jit_fns[variant];
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev < 64) cp->jit_devices.fetch_or(uint64_t(1) << dev);
        }
    }
    if (!jit_fns && (cp->fm != FM || cp->fs != FSLOTS || cp->outside)) {  // JIT unavailable: the interpreter's plan
        cp = compiled_plan(n, ops, nops, strict, reg_perm(flags & ~SVB_RUN_JIT), FM, FSLOTS, false);
        jit = false;
    }
    for (const PlanStep &st : cp->steps) {
        if (st.op >= 0) {
            single(st.mapped);
            continue;
        }
        const size_t pi = next_pass++;
        const FPass &P = cp->passes[pi];  // ~27 KiB, a __grid_constant__ kernel parameter
        const int64_t ntiles = n_amps >> P.fm;
        prof_begin(s);
        if (jit && jit_fns) {
            if (!jit_launch((*jit_fns)[pi], cp->passes[pi], a, ntiles, s)) {
                set_error("svb jit: cuLaunchKernel failed");
                return SVB_ECUDA;
            }
        } else if (fma) {
            k_fused<true><<<fused_grid(ntiles), FTHREADS, fused_smem(), s>>>(a, ntiles, P);
        } else {
            k_fused<false><<<fused_grid(ntiles), FTHREADS, fused_smem(), s>>>(a, ntiles, P);
        }
        prof_end(s, LaunchInfo{1, (jit && jit_fns) ? PROF_FUSED_JIT : PROF_FUSED, n_amps * 32});
        *launches += 1;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "k_fused launch");
    }
    return SVB_OK;
}

}  // namespace svb
