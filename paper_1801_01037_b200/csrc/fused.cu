// fused.cu -- op-list execution with multi-gate HBM passes.
//
// run_circuit applies one gate per sweep over the state (engine.py:483-494,
// _stride_cy.pyx:24-90): 7,800 full read+write passes for the configs[1]
// circuit.  Here a host-side planner (plan()) packs consecutive gates whose
// qubits fit in a set S of FM = 12 qubits into one pass; k_fused then
// streams the state tile by tile -- a tile is the 2^12 amplitudes that share
// all bits outside S -- through shared memory and applies every gate of the
// pass to it before writing it back: one HBM read + one write per pass.
//
//  * S always contains qubits 0..flow-1, so a tile is 2^(12-flow) runs of
//    2^flow contiguous amplitudes (flow = 4: 256 B runs) and every global
//    load/store is a coalesced 16 B-per-lane access.
//  * Loads are cp.async (LDGSTS, 16 B) into one of two 64 KiB tile buffers,
//    so tile i+1 streams in while tile i is computed (1 CTA of 512 threads
//    per SM, persistent over tiles).  Shared memory uses the 128 B XOR
//    swizzle phys(l) = l ^ ((l >> 3) & 7) so register-group reads are
//    bank-conflict free for any slot positions >= 3 or < 3 with lane spread.
//  * Gates are applied in "groups": each thread owns 8 amplitudes spanning 3
//    local bits (the group's slots); every non-diagonal gate of the group
//    targets a slot bit and runs entirely in registers; diagonal gates
//    (Z S T Rz CP) need no pairing and join any group; a control bit needs no
//    slot (it is a per-register or per-thread predicate).  Shared memory is
//    read and written once per group, not once per gate.
//  * Gate order: gates are applied in plan order with the exact single-gate
//    arithmetic (svb_common.cuh), so a strict-order plan is bit-identical to
//    op-by-op application.  The default plan may hoist a gate over earlier
//    gates on disjoint qubits (they commute); results then agree to a few ulp
//    (tested <= 1e-12, the north-star tolerance).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/svb.h"
#include "svb_common.cuh"

namespace svb {

LaunchInfo launch_gate(double2 *a, int64_t n_amps, const Gate &g, int t, int c, cudaStream_t s);

constexpr int FM = 12;                   // qubits per tile
constexpr int FTILE = 1 << FM;           // 4096 amplitudes = 64 KiB
constexpr int FTHREADS = FTILE / 8;      // 512 threads, 8 amplitudes each per group
constexpr int FMAXG = 160;               // gates per pass
constexpr int FMAXGRP = 80;              // register groups per pass
constexpr int FMAXROWS = FTILE / 8;      // rows when flow = 3

// Gate opcodes.  Non-diagonal: op = (kind * 3 + tslot) * 3 + cmode, kind in
// FK_*, tslot the register slot of the target, cmode 0 = no slot control,
// 1/2 = control on slot (tslot + cmode) % 3.  Diagonal: op = FOP_DIAG +
// (tpos * 4 + cpos) * 3 + var with tpos 0..2 = slot, 3 = a thread bit;
// cpos 0 = none, 1..3 = slot cpos-1; var 0 = general diag, 1 = q11 == 1,
// 2 = q11 == 1 and q22 in {+-1, +-i} (exact, no arithmetic).  A control on a
// thread bit (not a slot) is the per-thread predicate `cl`.
enum FKind { FK_GENERAL = 0, FK_REAL = 1, FK_ANTI = 2, FK_RX = 3, FK_UANTI = 4 };
constexpr int FOP_DIAG = 64;

struct FGate {
    double2 m[4];
    uint8_t op;
    int8_t tl;    // target local bit (diag with a thread-bit target)
    int8_t cl;    // control local bit when it is a thread bit, else -1
    uint8_t u;    // unit codes: bits 0-1 q12 (or q22 for diag), bits 2-3 q21
    int32_t pad;
};
struct FGroup {
    int8_t pos[3];  // local bits of the 3 register slots, ascending
    int8_t pad;
    int16_t first, count;
};
struct FPass {
    int ngates, ngroups, ncomp, flow;
    int8_t comp[64];        // tile-index bit j -> global qubit comp[j]
    int8_t rowbit[FM];      // local bit flow+j -> global qubit rowbit[j]
    FGroup groups[FMAXGRP];
    FGate gates[FMAXG];
};

__device__ __forceinline__ int swz(int l) { return l ^ ((l >> 3) & 7); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// x * u for u in {1, i, -1, -i} (code 0..3): exact, and equal to the
// reference's (ac - bd, ad + bc) with u's zero component (sign of 0 aside)
__device__ __forceinline__ double2 unit_mul(int code, double2 x) {
    double2 r = (code & 1) ? make_double2(-x.y, x.x) : x;
    return (code & 2) ? make_double2(-r.x, -r.y) : r;
}

template <int KIND, int S, int CS>
__device__ __forceinline__ void nd_gate(double2 (&v)[8], const FGate &fg) {
    Gate g;
    g.m[0] = fg.m[0];
    g.m[1] = fg.m[1];
    g.m[2] = fg.m[2];
    g.m[3] = fg.m[3];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i & (1 << S)) continue;
        if (CS >= 0 && !((i >> CS) & 1)) continue;
        double2 &lo = v[i];
        double2 &hi = v[i | (1 << S)];
        if (KIND == FK_UANTI) {
            double2 a = lo;
            lo = unit_mul(fg.u & 3, hi);
            hi = unit_mul((fg.u >> 2) & 3, a);
        } else if (KIND == FK_REAL) {
            pair_both<K_REAL>(g, lo, hi);
        } else if (KIND == FK_ANTI) {
            pair_both<K_ANTI>(g, lo, hi);
        } else if (KIND == FK_RX) {
            pair_both<K_RX>(g, lo, hi);
        } else {
            pair_both<K_GENERAL>(g, lo, hi);
        }
    }
}

template <int TP, int CP, int VAR>
__device__ __forceinline__ void diag_gate(double2 (&v)[8], const FGate &fg, int l0) {
    const bool tb = TP == 3 ? ((l0 >> fg.tl) & 1) : false;
    const double2 d0 = fg.m[0], d1 = fg.m[3];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (CP > 0 && !((i >> (CP - 1)) & 1)) continue;
        const bool b = TP == 3 ? tb : ((i >> TP) & 1);
        if (VAR == 0) {
            v[i] = cmul(b ? d1 : d0, v[i]);
        } else if (VAR == 1) {
            if (b) v[i] = cmul(d1, v[i]);
        } else {
            if (b) v[i] = unit_mul(fg.u & 3, v[i]);
        }
    }
}

#define SVB_ND3(K, S) \
    case ((K)*3 + (S)) * 3 + 0: nd_gate<K, S, -1>(v, fg); break; \
    case ((K)*3 + (S)) * 3 + 1: nd_gate<K, S, ((S) + 1) % 3>(v, fg); break; \
    case ((K)*3 + (S)) * 3 + 2: nd_gate<K, S, ((S) + 2) % 3>(v, fg); break;
#define SVB_ND(K) SVB_ND3(K, 0) SVB_ND3(K, 1) SVB_ND3(K, 2)
#define SVB_DG3(TP, CP) \
    case FOP_DIAG + ((TP)*4 + (CP)) * 3 + 0: diag_gate<TP, CP, 0>(v, fg, l0); break; \
    case FOP_DIAG + ((TP)*4 + (CP)) * 3 + 1: diag_gate<TP, CP, 1>(v, fg, l0); break; \
    case FOP_DIAG + ((TP)*4 + (CP)) * 3 + 2: diag_gate<TP, CP, 2>(v, fg, l0); break;
#define SVB_DG(TP) SVB_DG3(TP, 0) SVB_DG3(TP, 1) SVB_DG3(TP, 2) SVB_DG3(TP, 3)

__device__ __forceinline__ void run_gate(double2 (&v)[8], const FGate &fg, int l0) {
    switch (fg.op) {
        SVB_ND(FK_GENERAL)
        SVB_ND(FK_REAL)
        SVB_ND(FK_ANTI)
        SVB_ND(FK_RX)
        SVB_ND(FK_UANTI)
        SVB_DG(0)
        SVB_DG(1)
        SVB_DG(2)
        SVB_DG(3)
        default: break;
    }
}

__global__ void __launch_bounds__(FTHREADS, 1) k_fused(double2 *__restrict__ a, int64_t ntiles,
                                                       const __grid_constant__ FPass P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *tiles = reinterpret_cast<double2 *>(smem_raw);  // [2][FTILE]
    int64_t *rowoff = reinterpret_cast<int64_t *>(smem_raw + 2 * FTILE * sizeof(double2));
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

    auto tile_base = [&](int64_t tix) {
        int64_t b = 0;
        for (int j = 0; j < P.ncomp; ++j)
            if ((tix >> j) & 1) b |= int64_t(1) << P.comp[j];
        return b;
    };
    auto issue_load = [&](int64_t tix, double2 *buf) {
        const int64_t base = tile_base(tix);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int e = tid + k * FTHREADS;
            cp_async16(&buf[swz(e)], &a[base + rowoff[e >> flow] + (e & colmask)]);
        }
        cp_async_commit();
    };

    int64_t tix = blockIdx.x;
    if (tix < ntiles) issue_load(tix, tiles);
    for (int it = 0; tix < ntiles; ++it, tix += gridDim.x) {
        double2 *buf = tiles + (it & 1) * FTILE;
        cp_async_wait_all();
        __syncthreads();  // tile `tix` resident; previous tile's buffer free
        const int64_t next = tix + gridDim.x;
        if (next < ntiles) issue_load(next, tiles + ((it + 1) & 1) * FTILE);

        for (int gi = 0; gi < P.ngroups; ++gi) {
            const FGroup &G = P.groups[gi];
            const int p0 = G.pos[0], p1 = G.pos[1], p2 = G.pos[2];
            // thread's base local index: tid with zeros inserted at p0 < p1 < p2
            const int l0 = (int)insert_bit(insert_bit(insert_bit(tid, p0, 0), p1, 0), p2, 0);
            int li[8];
            double2 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                li[i] = l0 | ((i & 1) << p0) | (((i >> 1) & 1) << p1) | (((i >> 2) & 1) << p2);
                v[i] = buf[swz(li[i])];
            }
            const int qend = G.first + G.count;
            for (int q = G.first; q < qend; ++q) {
                const FGate &fg = P.gates[q];
                if (fg.cl >= 0 && !((l0 >> fg.cl) & 1)) continue;  // thread-bit control clear
                run_gate(v, fg, l0);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) buf[swz(li[i])] = v[i];
            __syncthreads();
        }

        const int64_t base = tile_base(tix);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int e = tid + k * FTHREADS;
            a[base + rowoff[e >> flow] + (e & colmask)] = buf[swz(e)];
        }
    }
    cp_async_wait_all();
}

// ---------------------------------------------------------------------------
// planner

struct PlanPass {
    uint64_t S = 0;  // global qubits in the tile
    std::vector<int> ops;
};

static int popc(uint64_t x) { return __builtin_popcountll(x); }

static int flow_bits() {
    static int f = [] {
        const char *e = getenv("SVB_FUSE_FLOW");
        int v = e ? atoi(e) : 4;
        return v < 3 ? 3 : (v > 5 ? 5 : v);
    }();
    return f;
}

static bool is_diag(const svb_op &o) {
    return o.q[2] == 0.0 && o.q[3] == 0.0 && o.q[4] == 0.0 && o.q[5] == 0.0;
}

static uint64_t op_mask(const svb_op &o) {
    uint64_t m = uint64_t(1) << o.target;
    if (o.kind == 1) m |= uint64_t(1) << o.control;
    return m;
}

// Greedy pass construction.  strict: only contiguous runs of ops.  Otherwise
// a scan over the remaining ops that hoists an op past skipped ones only if
// it shares no qubit with any skipped op (so every qubit keeps its order).
static std::vector<PlanPass> plan(int n, const svb_op *ops, int nops, bool strict) {
    std::vector<PlanPass> passes;
    const int flow = flow_bits();
    const uint64_t low = (uint64_t(1) << flow) - 1;
    std::vector<char> done(nops, 0);
    int first = 0;
    const int window = 4096;
    while (first < nops) {
        PlanPass p;
        p.S = low;
        uint64_t blocked = 0;
        int ngroups_est = 0;
        (void)ngroups_est;
        for (int i = first; i < nops && i < first + window; ++i) {
            if (done[i]) continue;
            uint64_t m = op_mask(ops[i]);
            bool fits = (m & blocked) == 0 && popc(p.S | m) <= FM && (int)p.ops.size() < FMAXG - 8;
            if (fits) {
                p.S |= m;
                p.ops.push_back(i);
                done[i] = 1;
            } else {
                if (strict) break;
                blocked |= m;
                if (popc(blocked | p.S) >= n) {
                    // every qubit is either in S or blocked: nothing later can join
                    bool any_free = false;
                    (void)any_free;
                }
            }
        }
        while (first < nops && done[first]) ++first;
        // pad S to exactly FM qubits (lowest unused qubits)
        for (int q = 0; q < n && popc(p.S) < FM; ++q) p.S |= uint64_t(1) << q;
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

struct GateMeta {
    Gate g;
    int tl, cl;  // local bits (cl = -1: none)
    bool diag;
};

// Build the kernel descriptor for one pass; false if it does not fit.
static bool build_pass(int n, const svb_op *ops, const PlanPass &pp, FPass &P) {
    memset(&P, 0, sizeof(P));
    P.flow = flow_bits();
    int local_of[64];
    int nl = 0, nc = 0;
    for (int q = 0; q < n; ++q) {
        if ((pp.S >> q) & 1) {
            local_of[q] = nl;
            if (nl >= P.flow) P.rowbit[nl - P.flow] = (int8_t)q;
            ++nl;
        } else {
            local_of[q] = -1;
            P.comp[nc++] = (int8_t)q;
        }
    }
    P.ncomp = nc;
    if ((int)pp.ops.size() > FMAXG) return false;
    std::vector<GateMeta> meta;
    for (int oi : pp.ops) {
        const svb_op &o = ops[oi];
        GateMeta m;
        m.g = make_gate(o.q);
        m.tl = local_of[o.target];
        m.cl = o.kind == 1 ? local_of[o.control] : -1;
        m.diag = m.g.kind == K_DIAG;
        meta.push_back(m);
    }
    // groups: consecutive gates whose non-diagonal targets use <= 3 slots
    int first = 0;
    const int ng = (int)meta.size();
    while (first < ng) {
        int slots[3], ns = 0, end = first;
        for (; end < ng; ++end) {
            if (meta[end].diag) continue;
            bool have = false;
            for (int i = 0; i < ns; ++i) have |= slots[i] == meta[end].tl;
            if (have) continue;
            if (ns == 3) break;
            slots[ns++] = meta[end].tl;
        }
        for (int b = FM - 1; ns < 3 && b >= 0; --b) {
            bool used = false;
            for (int i = 0; i < ns; ++i) used |= slots[i] == b;
            if (!used) slots[ns++] = b;
        }
        std::sort(slots, slots + 3);
        if (P.ngroups >= FMAXGRP) return false;
        FGroup &G = P.groups[P.ngroups++];
        for (int i = 0; i < 3; ++i) G.pos[i] = (int8_t)slots[i];
        G.first = (int16_t)first;
        G.count = (int16_t)(end - first);
        auto slot_of = [&](int l) {
            for (int i = 0; i < 3; ++i)
                if (slots[i] == l) return i;
            return -1;
        };
        for (int q = first; q < end; ++q) {
            const GateMeta &m = meta[q];
            FGate &fg = P.gates[q];
            for (int i = 0; i < 4; ++i) fg.m[i] = m.g.m[i];
            fg.tl = (int8_t)m.tl;
            fg.u = 0;
            int cs = m.cl >= 0 ? slot_of(m.cl) : -1;
            fg.cl = (int8_t)(m.cl >= 0 && cs < 0 ? m.cl : -1);
            if (m.diag) {
                int ts = slot_of(m.tl);
                int tpos = ts >= 0 ? ts : 3;
                int cpos = cs >= 0 ? cs + 1 : 0;
                int var = 0;
                if (m.g.d0_one) {
                    int uc = unit_code(m.g.m[3]);
                    var = uc >= 0 ? 2 : 1;
                    if (uc >= 0) fg.u = (uint8_t)uc;
                }
                fg.op = (uint8_t)(FOP_DIAG + (tpos * 4 + cpos) * 3 + var);
            } else {
                int ts = slot_of(m.tl);
                int kind;
                switch (m.g.kind) {
                    case K_REAL: kind = FK_REAL; break;
                    case K_ANTI: kind = FK_ANTI; break;
                    case K_RX: kind = FK_RX; break;
                    default: kind = FK_GENERAL; break;
                }
                if (m.g.kind == K_ANTI) {
                    int u12 = unit_code(m.g.m[1]), u21 = unit_code(m.g.m[2]);
                    if (u12 >= 0 && u21 >= 0) {
                        kind = FK_UANTI;
                        fg.u = (uint8_t)(u12 | (u21 << 2));
                    }
                }
                int cmode = cs >= 0 ? (cs - ts + 3) % 3 : 0;
                fg.op = (uint8_t)((kind * 3 + ts) * 3 + cmode);
            }
        }
        first = end;
    }
    P.ngates = ng;
    return true;
}

static size_t fused_smem() { return 2 * FTILE * sizeof(double2) + FMAXROWS * sizeof(int64_t); }

static int fused_grid(int64_t ntiles) {
    static int sms = [] {
        int d = 0, v = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        return v;
    }();
    return (int)std::min<int64_t>(ntiles, sms);
}

static bool fuse_enabled(int n, unsigned flags) {
    return (flags & SVB_RUN_FUSE) && n >= FM + 2;
}

int plan_passes(int n, const svb_op *ops, int nops, unsigned flags, int *groups) {
    if (groups) *groups = 0;
    if (!fuse_enabled(n, flags)) return nops;
    auto passes = plan(n, ops, nops, flags & SVB_RUN_STRICT_ORDER);
    if (groups) {
        FPass P;
        for (const PlanPass &pp : passes) {
            if (pp.ops.size() > 1 && build_pass(n, ops, pp, P)) *groups += P.ngroups;
        }
    }
    return (int)passes.size();
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem());
        attr_set = true;
    }
    auto passes = plan(n, ops, nops, flags & SVB_RUN_STRICT_ORDER);
    const int64_t ntiles = n_amps >> FM;
    FPass P;  // ~11 KiB, passed by value as a __grid_constant__ kernel parameter
    for (const PlanPass &pp : passes) {
        if (pp.ops.size() == 1) {
            single(ops[pp.ops[0]]);
            continue;
        }
        if (!build_pass(n, ops, pp, P)) {
            for (int oi : pp.ops) single(ops[oi]);
            continue;
        }
        prof_begin(s);
        k_fused<<<fused_grid(ntiles), FTHREADS, fused_smem(), s>>>(a, ntiles, P);
        prof_end(s, LaunchInfo{1, PROF_FUSED, n_amps * 32});
        *launches += 1;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "k_fused launch");
    }
    return SVB_OK;
}

}  // namespace svb
