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
constexpr int FMAXG = 144;               // gates per pass
constexpr int FMAXGRP = 64;              // register groups per pass
constexpr int FMAXROWS = FTILE / 8;      // rows when flow = 3

struct FGate {
    double2 m[4];
    int8_t kind, d0_one, diag, tslot, tl, cl, cslot, pad;
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

// apply one non-diagonal gate on register slot SLOT of the 8-amplitude block
template <int KIND, int SLOT>
__device__ __forceinline__ void reg_gate(double2 (&v)[8], const Gate &g, int cslot, bool thread_on) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i & (1 << SLOT)) continue;
        bool on = thread_on && (cslot < 0 || ((i >> cslot) & 1));
        if (on) pair_both<KIND>(g, v[i], v[i | (1 << SLOT)]);
    }
}

template <int KIND>
__device__ __forceinline__ void reg_gate_slot(double2 (&v)[8], const Gate &g, int slot, int cslot,
                                              bool thread_on) {
    if (slot == 0)
        reg_gate<KIND, 0>(v, g, cslot, thread_on);
    else if (slot == 1)
        reg_gate<KIND, 1>(v, g, cslot, thread_on);
    else
        reg_gate<KIND, 2>(v, g, cslot, thread_on);
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
            int l0 = (int)insert_bit(insert_bit(insert_bit(tid, p0, 0), p1, 0), p2, 0);
            int li[8];
            double2 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                li[i] = l0 | ((i & 1) << p0) | (((i >> 1) & 1) << p1) | (((i >> 2) & 1) << p2);
                v[i] = buf[swz(li[i])];
            }
            for (int q = G.first; q < G.first + G.count; ++q) {
                const FGate &fg = P.gates[q];
                Gate g;
                g.m[0] = fg.m[0];
                g.m[1] = fg.m[1];
                g.m[2] = fg.m[2];
                g.m[3] = fg.m[3];
                if (fg.diag) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        bool on = fg.cl < 0 || ((li[i] >> fg.cl) & 1);
                        bool b = (li[i] >> fg.tl) & 1;
                        if (on && (b || !fg.d0_one)) v[i] = cmul(b ? g.m[3] : g.m[0], v[i]);
                    }
                    continue;
                }
                bool thread_on = fg.cslot >= 0 || fg.cl < 0 || ((l0 >> fg.cl) & 1);
                switch (fg.kind) {
                    case K_REAL: reg_gate_slot<K_REAL>(v, g, fg.tslot, fg.cslot, thread_on); break;
                    case K_ANTI: reg_gate_slot<K_ANTI>(v, g, fg.tslot, fg.cslot, thread_on); break;
                    case K_RX: reg_gate_slot<K_RX>(v, g, fg.tslot, fg.cslot, thread_on); break;
                    default: reg_gate_slot<K_GENERAL>(v, g, fg.tslot, fg.cslot, thread_on); break;
                }
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

struct PlanGate {
    int op;  // index into ops
};
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

// Build the kernel descriptor for one pass; returns false if it needs > FMAXGRP groups.
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
    // groups: consecutive gates whose non-diagonal targets use <= 3 slots
    int g = 0;
    int cur_slots[3], nslots = 0;
    int grp_first = 0;
    bool overflow = false;
    auto close_group = [&](int upto) {
        if (upto == grp_first) return;
        if (P.ngroups >= FMAXGRP) {
            overflow = true;
            return;
        }
        FGroup &G = P.groups[P.ngroups++];
        // fill unused slots with the highest local bits not already used
        int s[3], k = 0;
        for (int i = 0; i < nslots; ++i) s[k++] = cur_slots[i];
        for (int b = FM - 1; k < 3 && b >= 0; --b) {
            bool used = false;
            for (int i = 0; i < k; ++i) used |= s[i] == b;
            if (!used) s[k++] = b;
        }
        std::sort(s, s + 3);
        for (int i = 0; i < 3; ++i) G.pos[i] = (int8_t)s[i];
        G.first = (int16_t)grp_first;
        G.count = (int16_t)(upto - grp_first);
        // resolve slots of this group's gates
        for (int q = grp_first; q < upto; ++q) {
            FGate &fg = P.gates[q];
            fg.tslot = fg.cslot = -1;
            for (int i = 0; i < 3; ++i) {
                if (s[i] == fg.tl) fg.tslot = (int8_t)i;
                if (fg.cl >= 0 && s[i] == fg.cl) fg.cslot = (int8_t)i;
            }
        }
        grp_first = upto;
        nslots = 0;
    };
    for (int oi : pp.ops) {
        const svb_op &o = ops[oi];
        Gate gg = make_gate(o.q);
        FGate &fg = P.gates[g];
        for (int i = 0; i < 4; ++i) fg.m[i] = gg.m[i];
        fg.kind = (int8_t)gg.kind;
        fg.d0_one = (int8_t)gg.d0_one;
        fg.diag = (int8_t)(gg.kind == K_DIAG);
        fg.tl = (int8_t)local_of[o.target];
        fg.cl = (int8_t)(o.kind == 1 ? local_of[o.control] : -1);
        if (!fg.diag) {
            bool have = false;
            for (int i = 0; i < nslots; ++i) have |= cur_slots[i] == fg.tl;
            if (!have) {
                if (nslots == 3) close_group(g);
                cur_slots[nslots++] = fg.tl;
            }
        }
        ++g;
    }
    P.ngates = g;
    close_group(g);
    return !overflow;
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

int plan_passes(int n, const svb_op *ops, int nops, unsigned flags) {
    if (!fuse_enabled(n, flags)) return nops;
    auto passes = plan(n, ops, nops, flags & SVB_RUN_STRICT_ORDER);
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
