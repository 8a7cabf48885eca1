// jit.cu -- runtime specialisation of fused passes (SVB_RUN_JIT).
//
// k_fused interprets a pass: a switch over opcode arms per gate, gate
// coefficients loaded from the parameter bank, per-register control masks
// tested at run time.  A circuit that runs many times (bench steps, parameter
// sweeps, VQE-style loops) can instead have each pass compiled once into
// straight-line code: coefficients become constant-bank operands, masks and
// slot patterns disappear at compile time, X/Y/S/S^dag become register
// renames, and ptxas can schedule arithmetic of consecutive gates together.
//
// The generated kernel has exactly the structure of k_fused (same tile,
// register groups, load/store maps, direct HBM groups, swizzle) and the same
// arithmetic (exact or FMA), so on the same plan its results equal the
// interpreter's bit for bit.  The fast variant (FMA + factor extraction, the
// bench default) adds what only generated code can do: tile-uniform
// predicates for qubits outside the tile, per-thread and per-slot phases,
// pending conditional swaps that gates pass through, a global factor applied
// by the circuit's last pass.  NVRTC compiles all passes of a plan in
// parallel host threads; loaded modules are shared by source hash and
// unloaded with the last plan using them.  tools/jit_emu.py runs the
// generated code on the host against the oracle (tests/test_jit_emu.py).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <memory>
#include <unordered_map>
#include <vector>

#include "fused_desc.h"

namespace svb {

namespace {

// slot bits / registers per thread of the pass being generated
thread_local int t_fs = FSLOTS;
inline int NS() { return t_fs; }
inline int NR() { return 1 << t_fs; }

struct Out {
    std::string s;
    __attribute__((format(printf, 2, 3))) void operator()(const char *fmt, ...) {
        char tmp[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(tmp, sizeof tmp, fmt, ap);
        va_end(ap);
        s += tmp;
    }
};

std::string hexf(double x) {
    char b[64];
    snprintf(b, sizeof b, "%a", x);
    return b;
}

// Gate coefficients live in a __constant__ table of the generated module:
// FP64 instructions take constant-bank operands directly, while literals
// would be materialised with two UMOVs each.  While a source is generated,
// lit() interns its value (by bit pattern) and names the table slot.
struct ConstPool {
    std::vector<double> vals;
    std::unordered_map<uint64_t, int> index;
};
thread_local ConstPool *t_pool = nullptr;

// a run of values at consecutive slots (tables indexed at run time): not interned
int pool_block(const std::vector<double> &v) {
    const int start = (int)t_pool->vals.size();
    t_pool->vals.insert(t_pool->vals.end(), v.begin(), v.end());
    return start;
}

std::string lit(double x) {
    if (!t_pool) return hexf(x);
    uint64_t bits;
    memcpy(&bits, &x, 8);
    auto it = t_pool->index.find(bits);
    int i;
    if (it != t_pool->index.end()) {
        i = it->second;
    } else {
        i = (int)t_pool->vals.size();
        t_pool->vals.push_back(x);
        t_pool->index[bits] = i;
    }
    return "kc[" + std::to_string(i) + "]";
}

const char *kPreamble = R"(
typedef long long i64;
struct alignas(16) d2 { double x, y; };
__device__ __forceinline__ d2 mk(double x, double y) { d2 r; r.x = x; r.y = y; return r; }
#if SVB_FMA
__device__ __forceinline__ d2 cm(double ar, double ai, d2 b) {   // (ar + i ai) * b
    return mk(__fma_rn(ar, b.x, -__dmul_rn(ai, b.y)), __fma_rn(ar, b.y, __dmul_rn(ai, b.x)));
}
__device__ __forceinline__ d2 row(double ar, double ai, d2 lo, double br, double bi, d2 hi) {
    return mk(__fma_rn(ar, lo.x, __fma_rn(-ai, lo.y, __fma_rn(br, hi.x, -__dmul_rn(bi, hi.y)))),
              __fma_rn(ar, lo.y, __fma_rn(ai, lo.x, __fma_rn(br, hi.y, __dmul_rn(bi, hi.x)))));
}
__device__ __forceinline__ d2 rrow(double a, d2 lo, double b, d2 hi) {
    return mk(__fma_rn(a, lo.x, __dmul_rn(b, hi.x)), __fma_rn(a, lo.y, __dmul_rn(b, hi.y)));
}
__device__ __forceinline__ d2 rirow(double a, d2 r, double s, d2 im) {  // a*r + (i s)*im
    return mk(__fma_rn(a, r.x, -__dmul_rn(s, im.y)), __fma_rn(a, r.y, __dmul_rn(s, im.x)));
}
#else
__device__ __forceinline__ d2 cm(double ar, double ai, d2 b) {
    return mk(__dsub_rn(__dmul_rn(ar, b.x), __dmul_rn(ai, b.y)), __dadd_rn(__dmul_rn(ar, b.y), __dmul_rn(ai, b.x)));
}
__device__ __forceinline__ d2 row(double ar, double ai, d2 lo, double br, double bi, d2 hi) {
    d2 p = cm(ar, ai, lo), q = cm(br, bi, hi);
    return mk(__dadd_rn(p.x, q.x), __dadd_rn(p.y, q.y));
}
__device__ __forceinline__ d2 rrow(double a, d2 lo, double b, d2 hi) {
    return mk(__dadd_rn(__dmul_rn(a, lo.x), __dmul_rn(b, hi.x)), __dadd_rn(__dmul_rn(a, lo.y), __dmul_rn(b, hi.y)));
}
__device__ __forceinline__ d2 rirow(double a, d2 r, double s, d2 im) {
    return mk(__dadd_rn(__dmul_rn(a, r.x), -__dmul_rn(s, im.y)), __dadd_rn(__dmul_rn(a, r.y), __dmul_rn(s, im.x)));
}
#endif
__device__ __forceinline__ void cpa(void *smem, const void *g) {
    unsigned s;
    asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(s) : "l"(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_u(unsigned s, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ unsigned su32(const void *p) {
    unsigned s;
    asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(s) : "l"(p));
    return s;
}
// tile ring (mode 3): one mbarrier per buffer counts the fill's cp.async
// completions (one no-increment arrival per issuing thread)
__device__ __forceinline__ void mb_init(unsigned long long *m, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(su32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive_cp(unsigned long long *m) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" :: "r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long *m, unsigned parity) {
    unsigned done;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(m)), "r"(parity) : "memory");
    } while (!done);
}
// barrier of one warpgroup (named barrier 1 + wg, its 128 threads)
__device__ __forceinline__ void wg_sync(int wg, int n) {
    asm volatile("bar.sync %0, %1;" :: "r"(wg + 1), "r"(n) : "memory");
}
__device__ __forceinline__ d2 ldcs(const d2 *p) {
    d2 r;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcs(d2 *p, d2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int swz(int l) { return l ^ ((l >> 3) ^ (l >> 6) ^ (l >> 9) ^ (l >> 12)) & 7; }
__device__ __forceinline__ double ng(double x) {  // -x as a sign-bit flip (integer pipe)
    return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ull);
}
__device__ __forceinline__ double cneg(double x, unsigned m) {  // -x where m = 0x80000000 (one LOP3)
    return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}
)";

int swz_h(int l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9) ^ (l >> 12)) & 7); }

unsigned xcombo_h(const uint32_t *s, int i) {
    unsigned r = 0;
    for (int k = 0; k < NS(); ++k)
        if ((i >> k) & 1) r ^= s[k];
    return r;
}
int64_t xcombo_g(const int64_t *s, int i) {
    int64_t r = 0;
    for (int k = 0; k < NS(); ++k)
        if ((i >> k) & 1) r ^= s[k];
    return r;
}
unsigned slot_pat(int s) {
    unsigned m = 0;
    for (int i = 0; i < NR(); ++i)
        if ((i >> s) & 1) m |= 1u << i;
    return m;
}

// predicate "bit b of the element's index is set" for a gate's thread-bit
// control / target (tid), or -- b >= FTILEBIT -- for a qubit outside the tile
// (a bit of the tile index tix: uniform over the CTA, a non-divergent branch)
std::string pbit(int b) {
    char buf[64];
    if (b >= FTILEBIT)
        snprintf(buf, sizeof buf, "((unsigned)(tix >> %d) & 1u)", b - FTILEBIT);
    else
        snprintf(buf, sizeof buf, "((tid >> %d) & 1)", b);
    return buf;
}

// one gate as straight-line code over v[0..15]
void emit_gate(Out &o, const FGate &g) {
    const double2 *m = g.m;
    const int op = g.op;
    const bool thread_ctl = g.cl >= 0;
    if (thread_ctl) o("if (%s) {\n", pbit(g.cl).c_str());
    if (op < FOP_DIAG) {
        const int kind = (op >> 1) / FSMAX, s = (op >> 1) % FSMAX, ctrl = op & 1;
        for (int i = 0; i < NR(); ++i) {
            if (i & (1 << s)) continue;
            if (ctrl && !((g.cmask >> i) & 1)) continue;
            const int j = i | (1 << s);
            o("{ const d2 L = v[%d], H = v[%d];\n", i, j);
            switch (kind) {
                case FK_REAL:
                    o("v[%d] = rrow(%s, L, %s, H); v[%d] = rrow(%s, L, %s, H); }\n", i, lit(m[0].x).c_str(),
                      lit(m[1].x).c_str(), j, lit(m[2].x).c_str(), lit(m[3].x).c_str());
                    break;
                case FK_RX:
                    o("v[%d] = rirow(%s, L, %s, H); v[%d] = rirow(%s, H, %s, L); }\n", i, lit(m[0].x).c_str(),
                      lit(m[1].y).c_str(), j, lit(m[3].x).c_str(), lit(m[2].y).c_str());
                    break;
                case FK_ANTI:
                    o("v[%d] = cm(%s, %s, H); v[%d] = cm(%s, %s, L); }\n", i, lit(m[1].x).c_str(),
                      lit(m[1].y).c_str(), j, lit(m[2].x).c_str(), lit(m[2].y).c_str());
                    break;
                default:
                    o("v[%d] = row(%s, %s, L, %s, %s, H); v[%d] = row(%s, %s, L, %s, %s, H); }\n", i,
                      lit(m[0].x).c_str(), lit(m[0].y).c_str(), lit(m[1].x).c_str(), lit(m[1].y).c_str(), j,
                      lit(m[2].x).c_str(), lit(m[2].y).c_str(), lit(m[3].x).c_str(), lit(m[3].y).c_str());
            }
        }
    } else {
        const int code = op - FOP_DIAG;
        const int ctrl = code & 1, tpos = (code >> 1) % (FSMAX + 1), var = (code >> 1) / (FSMAX + 1);
        auto mul = [&](int i, const double2 &d) {
            if (var == FD_Z && d.x == -1.0)
                o("v[%d] = mk(-v[%d].x, -v[%d].y);\n", i, i, i);
            else
                o("v[%d] = cm(%s, %s, v[%d]);\n", i, lit(d.x).c_str(), lit(d.y).c_str(), i);
        };
        const bool d0_one = var != FD_GENERAL;
        if (tpos == FTPOS_THREAD) {  // target on a thread bit: one factor per thread
            o("if (%s) {\n", pbit(g.tl).c_str());
            for (int i = 0; i < NR(); ++i)
                if (!ctrl || ((g.cmask >> i) & 1)) mul(i, m[3]);
            o("}");
            if (!d0_one) {
                o(" else {\n");
                for (int i = 0; i < NR(); ++i)
                    if (!ctrl || ((g.cmask >> i) & 1)) mul(i, m[0]);
                o("}");
            }
            o("\n");
        } else {
            for (int i = 0; i < NR(); ++i) {
                if (ctrl && !((g.cmask >> i) & 1)) continue;
                const bool b = (i >> tpos) & 1;
                if (b)
                    mul(i, m[3]);
                else if (!d0_one)
                    mul(i, m[0]);
            }
        }
    }
    if (thread_ctl) o("}\n");
}

// ---------------------------------------------------------------------------
// Unit-factor folding (FMA mode).  Gates whose entries are 0 / +-1 / +-i
// (X, Y, Z, S, S^dag, CZ, ...) do not need arithmetic: the generator keeps,
// per register, a pending factor u^c (u = i, c = 0..3) meaning "the
// amplitude is i^c times what the register holds".  A unit gate only
// renames registers and adds to c; the next arithmetic gate absorbs i^c into
// its coefficients (exact: multiplying a constant by +-1 / +-i swaps and
// negates its parts), with each product term in the same position of the
// same FMA chain as the interpreter's, so results equal the interpreter's up
// to the sign of zero.  Factors still pending when a group stores, or before
// a branch on the thread index, are applied with sign-bit flips (integer
// pipe, no DP instructions).

int unit_code(const double2 &z) {  // z = i^c -> c, else -1
    if (z.y == 0.0 && z.x == 1.0) return 0;
    if (z.x == 0.0 && z.y == 1.0) return 1;
    if (z.y == 0.0 && z.x == -1.0) return 2;
    if (z.x == 0.0 && z.y == -1.0) return 3;
    return -1;
}

// logical component `comp` (0 = re, 1 = im) of register `reg` named through
// the pending factor: returns the physical member and multiplies k's sign
const char *phys(int c, int comp, double &k) {
    // i^c (x + i y): c=0 (x, y)  c=1 (-y, x)  c=2 (-x, -y)  c=3 (y, -x)
    static const int member[4][2] = {{0, 1}, {1, 0}, {0, 1}, {1, 0}};
    static const int neg[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    if (neg[c][comp]) k = -k;
    return member[c][comp] ? "y" : "x";
}

struct Term {
    double k;
    const char *var;  // "L" / "H" / "X"
    int comp;         // logical component
    int code;         // pending factor of that register
};

// k0*t0 + (k1*t1 + (... + kn*tn)) as the interpreter's FMA chain
std::string chain(const std::vector<Term> &ts) {
    std::string e;
    for (int i = (int)ts.size() - 1; i >= 0; --i) {
        double k = ts[i].k;
        const char *m = phys(ts[i].code, ts[i].comp, k);
        char b[160];
        if (i == (int)ts.size() - 1)
            snprintf(b, sizeof b, "__dmul_rn(%s, %s.%s)", lit(k).c_str(), ts[i].var, m);
        else
            snprintf(b, sizeof b, "__fma_rn(%s, %s.%s, ", lit(k).c_str(), ts[i].var, m);
        e = (i == (int)ts.size() - 1) ? std::string(b) : std::string(b) + e + ")";
    }
    return e;
}

void materialize(Out &o, int *code, int i) {
    switch (code[i]) {
        case 1: o("v[%d] = mk(ng(v[%d].y), v[%d].x);\n", i, i, i); break;
        case 2: o("v[%d] = mk(ng(v[%d].x), ng(v[%d].y));\n", i, i, i); break;
        case 3: o("v[%d] = mk(v[%d].y, ng(v[%d].x));\n", i, i, i); break;
        default: break;
    }
    code[i] = 0;
}

// a*X for complex constant a (cm form): re = a.x X.x - a.y X.y, im = a.x X.y + a.y X.x
std::string cm_fold(const double2 &a, int cx) {
    return "mk(" + chain({{a.x, "X", 0, cx}, {-a.y, "X", 1, cx}}) + ", " +
           chain({{a.x, "X", 1, cx}, {a.y, "X", 0, cx}}) + ")";
}

// ---------------------------------------------------------------------------
// Pending conditional swaps (FMA modes).  A CNOT whose control is a thread
// bit and whose target is a slot swaps register pairs along that slot in
// half of the threads; done in place that is a divergent branch whose
// reconvergence costs 64 register moves.  Instead the generator records it
// (t_pend[slot] = thread bits whose parity says "swapped") and lets it ride:
// every later gate that pairs along another slot, is diagonal elsewhere, or
// is uniform per thread commutes with it; a gate that does not flushes it
// with branch-free selects; at the group's store the swap becomes a
// per-thread XOR of the store address (free).  Pending unit factors stay
// symmetric along a swapped slot, so they commute too.
// (mask bits 0-31: thread bits; 32-63: tile-index bits -- a CNOT controlled
// from outside the tile swaps the same way in every thread of some tiles)
thread_local uint64_t *t_pend = nullptr;

uint64_t pmask(int b) { return b >= FTILEBIT ? uint64_t(1) << (32 + b - FTILEBIT) : uint64_t(1) << b; }

std::string pcond(uint64_t m) {
    if ((m & (m - 1)) == 0) {
        int bit = 0;
        while (!((m >> bit) & 1)) ++bit;
        return pbit(bit >= 32 ? FTILEBIT + bit - 32 : bit);
    }
    const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
    char b[128];
    if (!hi)
        snprintf(b, sizeof b, "(__popc(tid & %uu) & 1)", lo);
    else if (!lo)
        snprintf(b, sizeof b, "(__popc((unsigned)tix & %uu) & 1)", hi);
    else
        snprintf(b, sizeof b, "((__popc(tid & %uu) ^ __popc((unsigned)tix & %uu)) & 1)", lo, hi);
    return b;
}

// pending unit factors of the group's registers (fast / fold modes): a flush
// swaps data, not codes, so a pair's codes must agree first (gates passed
// through a pending swap may leave them different)
thread_local int *t_code = nullptr;

void slot_phase_flush(Out &o, int s);

void pend_flush(Out &o, int s) {
    if (!t_pend || !t_pend[s]) return;
    slot_phase_flush(o, s);  // a data swap along s mixes its lo / hi registers
    if (t_code)
        for (int i = 0; i < NR(); ++i) {
            const int j = i | (1 << s);
            if (!(i & (1 << s)) && t_code[i] != t_code[j]) {
                materialize(o, t_code, i);
                materialize(o, t_code, j);
            }
        }
    o("{ const bool p = %s;\n", pcond(t_pend[s]).c_str());
    for (int i = 0; i < NR(); ++i) {
        if (i & (1 << s)) continue;
        const int j = i | (1 << s);
        o("{ const d2 a = v[%d], b = v[%d]; v[%d] = p ? b : a; v[%d] = p ? a : b; }\n", i, j, i, j);
    }
    o("}\n");
    t_pend[s] = 0;
}

int slot_of_mask(unsigned cmask, int t) {
    for (int k = 0; k < NS(); ++k) {
        unsigned pat = slot_pat(k) & ~(t >= 0 ? slot_pat(t) : 0u);
        if (k != t && pat == cmask) return k;
    }
    return -1;
}

// flush the pending swaps a gate does not commute with
void pend_conflicts(Out &o, const FGate &g) {
    if (!t_pend) return;
    const int op = g.op;
    if (op < FOP_DIAG) {
        const int t = (op >> 1) % FSMAX, ctrl = op & 1;
        // a gate of the form a I + b X on its target (X, CNOT, Rx, their
        // controlled forms) commutes with a pending swap on that slot
        const bool xtype = g.m[0].x == g.m[3].x && g.m[0].y == g.m[3].y && g.m[1].x == g.m[2].x &&
                           g.m[1].y == g.m[2].y;
        if (!xtype) pend_flush(o, t);
        if (ctrl) {
            const int k = slot_of_mask(g.cmask, t);
            if (k < 0)
                for (int x = 0; x < NS(); ++x) pend_flush(o, x);
            else
                pend_flush(o, k);
        }
    } else {
        const int c = op - FOP_DIAG;
        const int ctrl = c & 1, tpos = (c >> 1) % (FSMAX + 1);
        if (tpos < FTPOS_THREAD) pend_flush(o, tpos);
        if (ctrl) {
            const int k = slot_of_mask(g.cmask, -1);
            if (k < 0)
                for (int x = 0; x < NS(); ++x) pend_flush(o, x);
            else
                pend_flush(o, k);
        }
    }
}

void emit_gate_fold(Out &o, const FGate &g, int *code) {
    const double2 *m = g.m;
    const int op = g.op;
    const bool thread_ctl = g.cl >= 0;
    // CNOT from slot k to slot s while k has a pending swap X_k^p: since
    // X_k CNOT X_k = CNOT X_s, the registers get the plain CNOT (a rename)
    // and X_s^p joins the pending swaps -- no flush (exact data moves only)
    uint64_t carry = 0;
    int carry_to = -1;
    if (t_pend && op < FOP_DIAG && (op & 1) && !thread_ctl && m[0].x == 0 && m[0].y == 0 && m[3].x == 0 &&
        m[3].y == 0 && unit_code(m[1]) == 0 && unit_code(m[2]) == 0) {
        const int s = (op >> 1) % FSMAX;
        const int k = slot_of_mask(g.cmask, s);
        if (k >= 0 && t_pend[k]) {
            carry = t_pend[k];
            carry_to = s;
            t_pend[k] = 0;  // (kept out of pend_conflicts' flush)
        }
    }
    pend_conflicts(o, g);
    if (carry_to >= 0) {
        const int k = slot_of_mask(g.cmask, carry_to);
        t_pend[k] = carry;
    }
    if (op < FOP_DIAG) {
        const int kind = (op >> 1) / FSMAX, s = (op >> 1) % FSMAX, ctrl = op & 1;
        const int u12 = unit_code(m[1]), u21 = unit_code(m[2]);
        const bool unit_anti = m[0].x == 0.0 && m[0].y == 0.0 && m[3].x == 0.0 && m[3].y == 0.0 && u12 >= 0 &&
                               u21 >= 0;
        std::vector<int> lows;
        for (int i = 0; i < NR(); ++i) {
            if (i & (1 << s)) continue;
            if (ctrl && !((g.cmask >> i) & 1)) continue;
            lows.push_back(i);
        }
        if (thread_ctl && unit_anti && t_pend && u12 == 0 && u21 == 0 && !ctrl) {
            // controlled X on a thread-bit control: becomes a pending swap
            for (int i : lows) {
                const int j = i | (1 << s);
                if (code[i] != code[j]) {
                    materialize(o, code, i);
                    materialize(o, code, j);
                }
            }
            t_pend[s] ^= pmask(g.cl);
            return;
        }
        if (thread_ctl && unit_anti) {
            // controlled X / Y on a thread-bit control: a conditional swap (plus
            // sign flips for Y-like entries).  Equal pending factors on both
            // registers of a pair survive an X swap unchanged.
            for (int i : lows) {
                const int j = i | (1 << s);
                if (u12 != 0 || u21 != 0 || code[i] != code[j]) {
                    materialize(o, code, i);
                    materialize(o, code, j);
                }
            }
            o("if (%s) {\n", pbit(g.cl).c_str());
            for (int i : lows) {
                const int j = i | (1 << s);
                o("{ const d2 t = v[%d]; v[%d] = v[%d]; v[%d] = t; }\n", i, i, j, j);
                int tmp[FREGMAX] = {0};
                tmp[i] = u12;
                tmp[j] = u21;
                materialize(o, tmp, i);
                materialize(o, tmp, j);
            }
            o("}\n");
            return;
        }
        if (thread_ctl) {  // per-thread branch: pending factors must be uniform first
            for (int i : lows) {
                materialize(o, code, i);
                materialize(o, code, i | (1 << s));
            }
            o("if (%s) {\n", pbit(g.cl).c_str());
        }
        for (int i : lows) {
            const int j = i | (1 << s);
            const int cL = code[i], cH = code[j];
            if (unit_anti && !thread_ctl) {  // lo' = i^u12 hi, hi' = i^u21 lo: rename
                o("{ const d2 t = v[%d]; v[%d] = v[%d]; v[%d] = t; }\n", i, i, j, j);
                code[i] = (u12 + cH) & 3;
                code[j] = (u21 + cL) & 3;
                continue;
            }
            std::string lo, hi;
            switch (kind) {
                case FK_REAL:
                    lo = "mk(" + chain({{m[0].x, "L", 0, cL}, {m[1].x, "H", 0, cH}}) + ", " +
                         chain({{m[0].x, "L", 1, cL}, {m[1].x, "H", 1, cH}}) + ")";
                    hi = "mk(" + chain({{m[2].x, "L", 0, cL}, {m[3].x, "H", 0, cH}}) + ", " +
                         chain({{m[2].x, "L", 1, cL}, {m[3].x, "H", 1, cH}}) + ")";
                    break;
                case FK_RX:  // rirow(a, r, s, im) = (a r.x - s im.y, a r.y + s im.x)
                    lo = "mk(" + chain({{m[0].x, "L", 0, cL}, {-m[1].y, "H", 1, cH}}) + ", " +
                         chain({{m[0].x, "L", 1, cL}, {m[1].y, "H", 0, cH}}) + ")";
                    hi = "mk(" + chain({{m[3].x, "H", 0, cH}, {-m[2].y, "L", 1, cL}}) + ", " +
                         chain({{m[3].x, "H", 1, cH}, {m[2].y, "L", 0, cL}}) + ")";
                    break;
                case FK_ANTI:  // cm(q12, H), cm(q21, L)
                    lo = "mk(" + chain({{m[1].x, "H", 0, cH}, {-m[1].y, "H", 1, cH}}) + ", " +
                         chain({{m[1].x, "H", 1, cH}, {m[1].y, "H", 0, cH}}) + ")";
                    hi = "mk(" + chain({{m[2].x, "L", 0, cL}, {-m[2].y, "L", 1, cL}}) + ", " +
                         chain({{m[2].x, "L", 1, cL}, {m[2].y, "L", 0, cL}}) + ")";
                    break;
                default:  // row(a, L, b, H)
                    lo = "mk(" +
                         chain({{m[0].x, "L", 0, cL}, {-m[0].y, "L", 1, cL}, {m[1].x, "H", 0, cH},
                                {-m[1].y, "H", 1, cH}}) +
                         ", " +
                         chain({{m[0].x, "L", 1, cL}, {m[0].y, "L", 0, cL}, {m[1].x, "H", 1, cH},
                                {m[1].y, "H", 0, cH}}) +
                         ")";
                    hi = "mk(" +
                         chain({{m[2].x, "L", 0, cL}, {-m[2].y, "L", 1, cL}, {m[3].x, "H", 0, cH},
                                {-m[3].y, "H", 1, cH}}) +
                         ", " +
                         chain({{m[2].x, "L", 1, cL}, {m[2].y, "L", 0, cL}, {m[3].x, "H", 1, cH},
                                {m[3].y, "H", 0, cH}}) +
                         ")";
            }
            o("{ const d2 L = v[%d], H = v[%d];\nv[%d] = %s;\nv[%d] = %s; }\n", i, j, i, lo.c_str(), j, hi.c_str());
            code[i] = code[j] = 0;
        }
        if (thread_ctl) o("}\n");
        if (carry_to >= 0) t_pend[carry_to] ^= carry;
        return;
    }
    const int code_ = op - FOP_DIAG;
    const int ctrl = code_ & 1, tpos = (code_ >> 1) % (FSMAX + 1), var = (code_ >> 1) / (FSMAX + 1);
    const bool d0_one = var != FD_GENERAL;
    const bool branch = thread_ctl || tpos == FTPOS_THREAD;
    std::vector<int> regs;
    for (int i = 0; i < NR(); ++i)
        if (!ctrl || ((g.cmask >> i) & 1)) regs.push_back(i);
    auto mul = [&](int i, const double2 &d) {
        const int u = unit_code(d);
        if (u >= 0 && !branch) {
            code[i] = (code[i] + u) & 3;
            return;
        }
        if (u == 2) {  // -1 inside a branch: sign flips
            o("v[%d] = mk(ng(v[%d].x), ng(v[%d].y));\n", i, i, i);
            return;
        }
        o("{ const d2 X = v[%d]; v[%d] = %s; }\n", i, i, cm_fold(d, code[i]).c_str());
        code[i] = 0;
    };
    if (branch)
        for (int i : regs) materialize(o, code, i);
    if (thread_ctl) o("if (%s) {\n", pbit(g.cl).c_str());
    if (tpos == FTPOS_THREAD) {
        o("if (%s) {\n", pbit(g.tl).c_str());
        for (int i : regs) mul(i, m[3]);
        o("}");
        if (!d0_one) {
            o(" else {\n");
            for (int i : regs) mul(i, m[0]);
            o("}");
        }
        o("\n");
    } else {
        for (int i : regs) {
            if ((i >> tpos) & 1)
                mul(i, m[3]);
            else if (!d0_one)
                mul(i, m[0]);
        }
    }
    if (thread_ctl) o("}\n");
}

// ---------------------------------------------------------------------------
// Gates through a pending swap (fast mode).  A pending swap X^p on slot s
// (p: a per-thread / per-tile parity, see t_pend) need not be flushed before
// an uncontrolled gate G on s when X G X is G up to Pauli Z's and a sign:
// the registers then get G' = X^p G X^p and X^p stays pending --
//   X, Rx, unit anti-diagonal with q12 = q21 (X G X = G): nothing;
//   Y-like, q12 = -q21 (X G X = -G): ph *= (-1)^p;
//   Ry-like, q11 = q22, q12 = -q21 (X G X = Z G Z): Z^p before and after;
//   H-like, q11 = q12 = q21 = -q22 (H X = Z H): G, then Z^p, and the swap
//     is consumed;
//   diagonal (d0, d1): ph *= p ? d1 : d0, hi registers *= p ? d0/d1 : d1/d0.
// Z^p is a sign-bit XOR of the slot's hi registers; all of it costs a few
// integer ops instead of a select per register.
int pend_thru_mode() { return 31; }  // bits: 1 X-type, 2 Y-like, 4 Ry-like, 8 H-like, 16 diagonal
bool ceq(double2 a, double2 b) { return a.x == b.x && a.y == b.y; }
double2 cdivh(double2 a, double2 b);
double2 cnegh(double2 a) { return make_double2(-a.x, -a.y); }

void emit_phase(Out &o, const FGate &g);
extern thread_local bool t_phase;
void emit_gate_fast(Out &o, const FGate &g, int *code, double2 &F);

// sign flip of the hi registers of slot s where the mask's parity is odd
void emit_zp(Out &o, int s, uint64_t mask) {
    o("{ const unsigned pm = %s ? 0x80000000u : 0u;\n", pcond(mask).c_str());
    for (int i = 0; i < NR(); ++i)
        if ((i >> s) & 1) o("v[%d] = mk(cneg(v[%d].x, pm), cneg(v[%d].y, pm));\n", i, i, i);
    o("}\n");
}
extern thread_local bool t_phase_sign;
extern thread_local unsigned t_hs;
void emit_phase_sign(Out &o, uint64_t mask) {  // ph *= (-1)^p
    o("{ const unsigned pm = %s ? 0x80000000u : 0u; ph = mk(cneg(ph.x, pm), cneg(ph.y, pm)); }\n",
      pcond(mask).c_str());
    if (!t_phase) t_phase_sign = true;  // (ph stays +-1 unless a phase joins)
    t_phase = true;
}

bool pend_through(Out &o, const FGate &g, int *code, double2 &F) {
    const int pt = pend_thru_mode();
    if (!t_pend || !pt || g.cl >= 0 || (g.op & 1)) return false;
    const double2 *m = g.m;
    if (g.op < FOP_DIAG) {
        const int s = (g.op >> 1) % FSMAX;
        const uint64_t mask = t_pend[s];
        if (!mask) return false;
        const bool xtype = ceq(m[0], m[3]) && ceq(m[1], m[2]);
        const bool ylike = m[0].x == 0 && m[0].y == 0 && m[3].x == 0 && m[3].y == 0 && ceq(m[1], cnegh(m[2])) &&
                           unit_code(m[1]) >= 0;
        const bool rylike = ceq(m[0], m[3]) && ceq(m[1], cnegh(m[2])) && !ylike;
        const bool hlike = ceq(m[0], m[1]) && ceq(m[0], m[2]) && ceq(m[0], cnegh(m[3]));
        if (!((xtype && (pt & 1)) || (ylike && (pt & 2)) || (rylike && (pt & 4)) || (hlike && (pt & 8))))
            return false;
        t_pend[s] = 0;  // emit G itself without flushing s
        if (rylike) emit_zp(o, s, mask);
        emit_gate_fast(o, g, code, F);
        if (rylike) emit_zp(o, s, mask);
        if (hlike) {
            emit_zp(o, s, mask);
            return true;  // consumed
        }
        if (ylike) emit_phase_sign(o, mask);
        t_pend[s] = mask;
        return true;
    }
    const int c = g.op - FOP_DIAG;
    const int tpos = (c >> 1) % (FSMAX + 1);
    if (tpos >= FTPOS_THREAD || !t_pend[tpos] || !(pt & 16)) return false;
    const int s = tpos;
    const uint64_t mask = t_pend[s];
    const double2 d0 = m[0], d1 = m[3];
    if ((d0.x == 0 && d0.y == 0) || (d1.x == 0 && d1.y == 0)) return false;
    const double2 r = cdivh(d1, d0), ri = cdivh(d0, d1);
    // ph *= p ? d1 : d0
    o("{ const bool p = %s;\n", pcond(mask).c_str());
    o("ph = cm(p ? %s : %s, p ? %s : %s, ph);\n", lit(d1.x).c_str(), lit(d0.x).c_str(), lit(d1.y).c_str(),
      lit(d0.y).c_str());
    t_phase = true;
    t_phase_sign = false;
    const int ur = unit_code(r), uri = unit_code(ri);
    if (ur >= 0 && uri >= 0) {
        // r = i^u, 1/r = i^-u = i^u (-1)^[u odd]: a code plus a conditional sign
        const bool odd = ur & 1;
        for (int i = 0; i < NR(); ++i)
            if ((i >> s) & 1) code[i] = (code[i] + ur) & 3;
        if (odd) {
            o("const unsigned pm = p ? 0x80000000u : 0u;\n");
            for (int i = 0; i < NR(); ++i)
                if ((i >> s) & 1) o("v[%d] = mk(cneg(v[%d].x, pm), cneg(v[%d].y, pm));\n", i, i, i);
        }
    } else {
        // the hi registers' factor p ? 1/r : r joins slot s's per-slot phase
        // (applied once, merged with the group-end multiply when there is one)
        o("hs%d = cm(p ? %s : %s, p ? %s : %s, hs%d);\n", s, lit(ri.x).c_str(), lit(r.x).c_str(),
          lit(ri.y).c_str(), lit(r.y).c_str(), s);
        t_hs |= 1u << s;
    }
    o("}\n");
    return true;
}

// ---------------------------------------------------------------------------
// Factor extraction ("fast" FMA mode, SVB_JIT_FACTOR, default on).  An
// uncontrolled one-qubit gate multiplies EVERY amplitude of the state, so a
// scalar can be pulled out of it: U = a V with one entry of V equal to 1
// (H = s [[1,1],[1,-1]], Ry = c [[1,-t],[t,1]], Rx = c [[1,-it],[-it,1]],
// Rz = e^{-i th/2} diag(1, e^{i th})).  The pass applies V -- one FMA or add
// per output part instead of a multiply and an FMA -- and the generator
// multiplies a into a global factor F that the state carries: stored =
// true / F.  F is applied (one complex multiply per amplitude) at the end of
// the last fused pass of the circuit, or earlier when |F| leaves
// [2^-200, 2^200].  Everything else the state meets in between (single-gate
// kernels, controlled gates) is linear, so it commutes with the scalar.
// Rounding differs from the reference at the 1e-16 level (within the FMA
// mode's 1e-12 tolerance); exact and strict modes never extract.

bool jit_factor_on() {
    const char *e = getenv("SVB_JIT_FACTOR");
    return e ? atoi(e) != 0 : true;
}

double2 cmulh(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
double2 cdivh(double2 a, double2 b) {
    if (b.y == 0.0) return make_double2(a.x / b.x, a.y / b.x);
    const double d = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
double cabsh(double2 a) { return std::hypot(a.x, a.y); }

struct FTerm {
    double k;
    const char *var;
    int comp;  // logical component of var
    int code;  // pending unit factor of var's register
};

// sum of k * var.comp with zero terms dropped and +-1 terms added plainly
std::string fast_sum(const std::vector<FTerm> &ts) {
    std::vector<std::pair<double, std::string>> unit, other;
    for (const FTerm &t : ts) {
        if (t.k == 0.0) continue;
        double k = t.k;
        const char *m = phys(t.code, t.comp, k);
        std::string v = std::string(t.var) + "." + m;
        if (k == 1.0 || k == -1.0)
            unit.push_back({k, v});
        else
            other.push_back({k, v});
    }
    std::string e;
    if (!unit.empty()) {
        e = (unit[0].first < 0 ? "-" : "") + unit[0].second;
        for (size_t i = 1; i < unit.size(); ++i)
            e = "__dadd_rn(" + e + ", " + (unit[i].first < 0 ? "-" : "") + unit[i].second + ")";
    }
    for (size_t i = 0; i < other.size(); ++i) {
        if (e.empty())
            e = "__dmul_rn(" + lit(other[i].first) + ", " + other[i].second + ")";
        else
            e = "__fma_rn(" + lit(other[i].first) + ", " + other[i].second + ", " + e + ")";
    }
    return e.empty() ? std::string("0.0") : e;
}

// DP instructions fast_sum needs for one output part with the given weights
int part_cost(std::initializer_list<double> ks) {
    int n = 0, u = 0;
    for (double k : ks)
        if (k != 0.0) {
            ++n;
            u += (k == 1.0 || k == -1.0);
        }
    return n == 0 ? 0 : (u ? n - 1 : n);
}

// a L + b H, both parts
std::string lin2(double2 a, int cL, double2 b, int cH) {
    return "mk(" +
           fast_sum({{a.x, "L", 0, cL}, {-a.y, "L", 1, cL}, {b.x, "H", 0, cH}, {-b.y, "H", 1, cH}}) + ", " +
           fast_sum({{a.x, "L", 1, cL}, {a.y, "L", 0, cL}, {b.x, "H", 1, cH}, {b.y, "H", 0, cH}}) + ")";
}
int lin2_cost(double2 a, double2 b) {
    return part_cost({a.x, -a.y, b.x, -b.y}) + part_cost({a.x, a.y, b.x, b.y});
}

// choose the scalar to pull out of a 2x2 (all four entries as candidates,
// plus none); only well-conditioned ones (|a| >= 0.7 max |entry|)
double2 pick_factor(const double2 *m, bool diag) {
    double mx = 0;
    for (int i = 0; i < 4; ++i) mx = std::max(mx, cabsh(m[i]));
    double2 best = make_double2(1.0, 0.0);
    auto cost_of = [&](double2 a) {
        double2 v[4];
        for (int i = 0; i < 4; ++i) v[i] = cdivh(m[i], a);
        if (diag) return lin2_cost(v[0], make_double2(0, 0)) + lin2_cost(make_double2(0, 0), v[3]);
        return lin2_cost(v[0], v[1]) + lin2_cost(v[2], v[3]);
    };
    int best_cost = cost_of(best);
    for (int i = 0; i < 4; ++i) {
        if (cabsh(m[i]) < 0.7 * mx || cabsh(m[i]) == 0.0) continue;
        const int c = cost_of(m[i]);
        if (c < best_cost) {
            best_cost = c;
            best = m[i];
        }
    }
    return best;
}

// Per-thread phase (fast mode).  A diagonal gate whose target and control
// (if any) are thread or tile bits multiplies ALL registers of a thread by
// one scalar; such scalars commute with every in-register gate, so the
// generator multiplies them into a per-thread `ph` (a few scalar
// instructions per gate instead of a predicated multiply of every register)
// and applies ph once, at the end of the group, fused with the global
// factor when that is due.
// (Found with it: the last-pass flag was shadowed by the last-group flag, so
// F was applied at the end of every pass -- exact, but one multiply of every
// register per pass; now only the circuit's last pass applies it.)
thread_local bool t_phase = false;  // the current group's ph is not 1
thread_local bool t_phase_sign = false;  // ... and it is only a sign, +-1

int phase_mode() { return 7; }  // bits: 1 thread targets, 2 tile targets, 4 controlled

// ph *= (target bit ? d1 : d0), under the (thread / tile) control if any
// Tile-uniform phase factors of a group, merged.  A controlled phase whose
// phase-carrying bit is a tile bit (a qubit outside the tile) multiplies ph by
// a value every thread of the tile computes alike; the QFT's passes carry
// chains of ~18 of them per thread-bit qubit (a complex multiply and two
// selects each: 100 in QFT-30's first pass, a fifth of its instructions).
// They all commute with everything until ph is applied at the group's end,
// so they are collected per thread condition and emitted there as products
// looked up in small tables: up to five tile bits index a 32-entry table of
// precomputed products in the constant bank (a uniform load), one complex
// multiply per table instead of one per gate.  SVB_JIT_TPH=0 keeps one
// multiply per gate (measurement).
struct TilePhase {
    uint32_t mask;  // tile-index bits that must all be set
    int cond;       // thread bit that must be set too, -1: none
    double2 d;
};
thread_local std::vector<TilePhase> *t_tph = nullptr;
// the same for per-slot phases hs<s> (a controlled phase between slot s and a
// qubit outside the tile): factor f1 where the tile bit is set, f0 where not
struct SlotTilePhase {
    int bit;
    double2 f1, f0;
};
thread_local std::vector<SlotTilePhase> *t_shs = nullptr;  // [slot]

void materialize_slot_tile(Out &o, int s);

bool tph_on() {
    static const bool on = [] {
        const char *e = getenv("SVB_JIT_TPH");
        return !e || atoi(e) != 0;
    }();
    return on;
}

void flush_tile_phases(Out &o) {
    if (!t_tph || t_tph->empty()) return;
    std::vector<int> conds;
    for (const TilePhase &f : *t_tph)
        if (std::find(conds.begin(), conds.end(), f.cond) == conds.end()) conds.push_back(f.cond);
    for (int c : conds) {
        std::vector<TilePhase> fs;
        for (const TilePhase &f : *t_tph)
            if (f.cond == c) fs.push_back(f);
        std::vector<char> done(fs.size(), 0);
        for (size_t i = 0; i < fs.size(); ++i) {
            if (done[i]) continue;
            // grow a chunk of at most five tile bits from the unplaced factors, in order
            uint32_t bits = 0;
            std::vector<size_t> in;
            for (size_t j = i; j < fs.size(); ++j) {
                if (done[j]) continue;
                if (__builtin_popcount(bits | fs[j].mask) > 5) continue;
                bits |= fs[j].mask;
                in.push_back(j);
                done[j] = 1;
            }
            std::vector<int> pos;
            for (int b = 0; b < 32; ++b)
                if ((bits >> b) & 1) pos.push_back(b);
            const int nb = (int)pos.size();
            std::vector<double> tab;
            for (int ix = 0; ix < (1 << nb); ++ix) {
                uint32_t set = 0;
                for (int k = 0; k < nb; ++k)
                    if ((ix >> k) & 1) set |= 1u << pos[k];
                double2 v = make_double2(1.0, 0.0);
                for (size_t j : in)
                    if ((fs[j].mask & set) == fs[j].mask) v = cmulh(v, fs[j].d);
                tab.push_back(v.x);
                tab.push_back(v.y);
            }
            const int start = pool_block(tab);
            o("{ const unsigned ix = 0u");
            for (int k = 0; k < nb; ++k) o(" | (((unsigned)(tix >> %d) & 1u) << %d)", pos[k], k);
            o(";\n");
            if (c < 0)
                o("ph = cm(kc[%d + 2 * ix], kc[%d + 2 * ix], ph);\n", start, start + 1);
            else  // branch-free, like emit_phase
                o("{ const bool b = %s; ph = cm(b ? kc[%d + 2 * ix] : 1.0, b ? kc[%d + 2 * ix] : 0.0, ph); }\n",
                  pbit(c).c_str(), start, start + 1);
            o("}\n");
        }
    }
    t_tph->clear();
}

// multiply slot s's collected tile-uniform factors into hs<s> (before hs<s> is read)
void materialize_slot_tile(Out &o, int s) {
    if (!t_shs || t_shs[s].empty()) return;
    std::vector<SlotTilePhase> &fs = t_shs[s];
    std::vector<char> done(fs.size(), 0);
    for (size_t i = 0; i < fs.size(); ++i) {
        if (done[i]) continue;
        uint32_t bits = 0;
        std::vector<size_t> in;
        for (size_t j = i; j < fs.size(); ++j) {
            if (done[j]) continue;
            if (__builtin_popcount(bits | (1u << fs[j].bit)) > 5) continue;
            bits |= 1u << fs[j].bit;
            in.push_back(j);
            done[j] = 1;
        }
        std::vector<int> pos;
        for (int b = 0; b < 32; ++b)
            if ((bits >> b) & 1) pos.push_back(b);
        const int nb = (int)pos.size();
        std::vector<double> tab;
        for (int ix = 0; ix < (1 << nb); ++ix) {
            uint32_t set = 0;
            for (int k = 0; k < nb; ++k)
                if ((ix >> k) & 1) set |= 1u << pos[k];
            double2 v = make_double2(1.0, 0.0);
            for (size_t j : in) v = cmulh(v, ((set >> fs[j].bit) & 1) ? fs[j].f1 : fs[j].f0);
            tab.push_back(v.x);
            tab.push_back(v.y);
        }
        const int start = pool_block(tab);
        o("{ const unsigned ix = 0u");
        for (int k = 0; k < nb; ++k) o(" | (((unsigned)(tix >> %d) & 1u) << %d)", pos[k], k);
        o("; hs%d = cm(kc[%d + 2 * ix], kc[%d + 2 * ix], hs%d); }\n", s, start, start + 1, s);
    }
    fs.clear();
}

void emit_phase(Out &o, const FGate &g) {
    const double2 d0 = g.m[0], d1 = g.m[3];
    const bool one0 = unit_code(d0) == 0;
    if (t_tph && t_pool && one0 && tph_on()) {
        // phase d1 where every bit of the gate is set; at least one of them a tile bit
        const bool tt = g.tl >= FTILEBIT, ct = g.cl >= FTILEBIT;
        TilePhase f;
        f.d = d1;
        f.mask = 0;
        f.cond = -1;
        bool ok = false;
        if (tt && g.tl - FTILEBIT < 32) {
            f.mask = 1u << (g.tl - FTILEBIT);
            if (g.cl < 0) {
                ok = true;
            } else if (ct && g.cl - FTILEBIT < 32) {
                f.mask |= 1u << (g.cl - FTILEBIT);
                ok = true;
            } else if (!ct) {
                f.cond = g.cl;
                ok = true;
            }
        } else if (!tt && ct && g.cl - FTILEBIT < 32) {
            f.mask = 1u << (g.cl - FTILEBIT);
            f.cond = g.tl;
            ok = true;
        }
        if (ok) {
            t_tph->push_back(f);
            t_phase = true;
            t_phase_sign = false;
            return;
        }
    }
    o("{ const bool b = %s;\n", pbit(g.tl).c_str());
    if (g.cl >= 0) o("if (%s) {\n", pbit(g.cl).c_str());
    // branch-free (a predicated update of ph is miscompiled by ptxas -O1+ in
    // some long passes -- found by tools/jit_emu.py agreeing with the oracle
    // while the device did not, and ptxas -O0 agreeing)
    if (one0)
        o("ph = cm(b ? %s : 1.0, b ? %s : 0.0, ph);\n", lit(d1.x).c_str(), lit(d1.y).c_str());
    else
        o("ph = cm(b ? %s : %s, b ? %s : %s, ph);\n", lit(d1.x).c_str(), lit(d0.x).c_str(), lit(d1.y).c_str(),
          lit(d0.y).c_str());
    if (g.cl >= 0) o("}\n");
    o("}\n");
    t_phase = true;
    t_phase_sign = false;
}

// ph * (i^c X) for register X holding a pending unit factor c
std::string cm_ph(int c) {
    double k1 = 1.0, k2 = 1.0;
    const char *m1 = phys(c, 0, k1), *m2 = phys(c, 1, k2);
    auto sg = [](double k) { return k < 0 ? "-" : ""; };
    char b[256];
    snprintf(b, sizeof b, "mk(__fma_rn(ph.x, %sX.%s, %s__dmul_rn(ph.y, X.%s)), __fma_rn(ph.x, %sX.%s, %s__dmul_rn(ph.y, X.%s)))",
             sg(k1), m1, sg(-k2), m2, sg(k2), m2, sg(k1), m1);
    return b;
}

// Per-slot phases (fast mode).  A diagonal gate whose only slot is s --
// target s under a thread / tile control with q11 = 1 (controlled phase
// from a thread or a qubit outside the tile), or control s with a thread /
// tile target -- multiplies the registers with slot bit s set by one
// per-thread value.  Those values are multiplied into a per-thread `hs<s>`
// (scalar work) and applied to the 16 registers once, when a non-diagonal
// gate targets s, a pending swap along s is flushed, or the group ends:
// QFT passes carry dozens of such phases per slot.
thread_local unsigned t_hs = 0;  // slots whose hs is not 1

// Pending constant diagonals (fast mode).  An uncontrolled diagonal gate on
// slot s, diag(1, d) after factor extraction with d not a unit, multiplies
// the 16 registers with slot bit s set by the compile-time constant d.  It
// commutes with every gate that does not target s (a pair update along
// another slot sees the same factor on both registers of a pair; controls
// on s select whole halves), so it is kept pending as t_pd[s] -- further
// diagonals on s multiply into it -- and applied when a gate targets s or
// at the group's end, where each register's pending constants ride on the
// per-thread phase or the global factor that is applied anyway (one
// complex multiply per register for all of them).
thread_local double2 t_pd[FSMAX];
thread_local unsigned t_pdm = 0;  // slots with a pending constant

void pd_flush(Out &o, int s);

bool slot_phase_on() { return true; }

void slot_phase_flush(Out &o, int s) {
    if (!((t_hs >> s) & 1) || !t_code) return;
    materialize_slot_tile(o, s);
    for (int i = 0; i < NR(); ++i) {
        if (!((i >> s) & 1)) continue;
        double k1 = 1.0, k2 = 1.0;
        const char *m1 = phys(t_code[i], 0, k1), *m2 = phys(t_code[i], 1, k2);
        auto sg = [](double k) { return k < 0 ? "-" : ""; };
        o("{ const d2 X = v[%d]; v[%d] = mk(__fma_rn(hs%d.x, %sX.%s, %s__dmul_rn(hs%d.y, X.%s)), "
          "__fma_rn(hs%d.x, %sX.%s, %s__dmul_rn(hs%d.y, X.%s))); }\n",
          i, i, s, sg(k1), m1, sg(-k2), s, m2, s, sg(k2), m2, sg(k1), s, m1);
        t_code[i] = 0;
    }
    o("hs%d = mk(1.0, 0.0);\n", s);
    t_hs &= ~(1u << s);
}

// true if g was taken into a per-slot phase
bool slot_phase_take(Out &o, const FGate &g) {
    if (g.op < FOP_DIAG || !slot_phase_on()) return false;
    const int c = g.op - FOP_DIAG;
    const int tpos = (c >> 1) % (FSMAX + 1);
    int s;
    std::string pred;
    double2 f1, f0;  // factor when pred holds / not
    if (tpos < FTPOS_THREAD && !(c & 1) && g.cl >= 0 && unit_code(g.m[0]) == 0) {
        s = tpos;  // target slot, thread / tile control
        pred = pbit(g.cl);
        f1 = g.m[3];
        f0 = make_double2(1.0, 0.0);
    } else if (tpos == FTPOS_THREAD && (c & 1) && g.cl < 0) {
        s = slot_of_mask(g.cmask, -1);  // control slot, thread / tile target
        if (s < 0) return false;
        pred = pbit(g.tl);
        f1 = g.m[3];
        f0 = g.m[0];
    } else {
        return false;
    }
    if (t_pend && t_pend[s]) return false;  // (the pending-swap paths handle it)
    {
        const int pb = (tpos < FTPOS_THREAD) ? g.cl : g.tl;  // the predicate's bit
        if (t_shs && t_pool && tph_on() && pb >= FTILEBIT && pb - FTILEBIT < 32) {
            t_shs[s].push_back(SlotTilePhase{pb - FTILEBIT, f1, f0});
            t_hs |= 1u << s;
            return true;
        }
    }
    o("{ const bool b = %s; hs%d = cm(b ? %s : %s, b ? %s : %s, hs%d); }\n", pred.c_str(), s, lit(f1.x).c_str(),
      lit(f0.x).c_str(), lit(f1.y).c_str(), lit(f0.y).c_str(), s);
    t_hs |= 1u << s;
    return true;
}

bool pend_through(Out &o, const FGate &g, int *code, double2 &F);

void emit_gate_fast(Out &o, const FGate &g, int *code, double2 &F) {
    const int op = g.op;
    if (slot_phase_take(o, g)) return;
    if (op < FOP_DIAG) {  // a non-diagonal gate on that slot
        slot_phase_flush(o, (op >> 1) % FSMAX);
        pd_flush(o, (op >> 1) % FSMAX);
    }
    if (pend_through(o, g, code, F)) return;
    if (op >= FOP_DIAG && phase_mode()) {
        const int c = op - FOP_DIAG, pm = phase_mode();
        const bool ok = ((g.tl >= FTILEBIT) ? (pm & 2) : (pm & 1)) && (g.cl < 0 || (pm & 4));
        if (ok && !(c & 1) && (c >> 1) % (FSMAX + 1) == FTPOS_THREAD) {  // scalar per thread
            emit_phase(o, g);
            return;
        }
    }
    const bool uncontrolled = g.cl < 0 && !(op & 1);
    if (!uncontrolled) {  // a controlled gate scales only part of the state
        emit_gate_fold(o, g, code);  // (handles the pending swaps itself)
        return;
    }
    pend_conflicts(o, g);
    if (op < FOP_DIAG) {
        const int s = (op >> 1) % FSMAX;
        const int u12 = unit_code(g.m[1]), u21 = unit_code(g.m[2]);
        if (g.m[0].x == 0.0 && g.m[0].y == 0.0 && g.m[3].x == 0.0 && g.m[3].y == 0.0 && u12 >= 0 && u21 >= 0) {
            emit_gate_fold(o, g, code);  // a pure rename already
            return;
        }
        const double2 a = pick_factor(g.m, false);
        double2 v[4];
        for (int i = 0; i < 4; ++i) v[i] = cdivh(g.m[i], a);
        F = cmulh(F, a);
        for (int i = 0; i < NR(); ++i) {
            if (i & (1 << s)) continue;
            const int j = i | (1 << s);
            o("{ const d2 L = v[%d], H = v[%d];\nv[%d] = %s;\nv[%d] = %s; }\n", i, j, i,
              lin2(v[0], code[i], v[1], code[j]).c_str(), j, lin2(v[2], code[i], v[3], code[j]).c_str());
            code[i] = code[j] = 0;
        }
        return;
    }
    const int c = op - FOP_DIAG;
    const int tpos = (c >> 1) % (FSMAX + 1);
    const double2 a = pick_factor(g.m, true);
    const double2 d0 = cdivh(g.m[0], a), d1 = cdivh(g.m[3], a);
    F = cmulh(F, a);
    auto mul = [&](int i, double2 d, bool branch) {
        const int u = unit_code(d);
        if (u >= 0 && !branch) {
            code[i] = (code[i] + u) & 3;
            return;
        }
        o("{ const d2 X = v[%d]; v[%d] = mk(%s, %s); }\n", i, i,
          fast_sum({{d.x, "X", 0, code[i]}, {-d.y, "X", 1, code[i]}}).c_str(),
          fast_sum({{d.x, "X", 1, code[i]}, {d.y, "X", 0, code[i]}}).c_str());
        code[i] = 0;
    };
    if (tpos == FTPOS_THREAD) {  // target on a thread bit: the factor depends on the thread
        const bool one0 = unit_code(d0) == 0, one1 = unit_code(d1) == 0;
        for (int i = 0; i < NR(); ++i) materialize(o, code, i);
        if (!one1) {
            o("if (%s) {\n", pbit(g.tl).c_str());
            for (int i = 0; i < NR(); ++i) mul(i, d1, true);
            o("}\n");
        }
        if (!one0) {
            o("if (!%s) {\n", pbit(g.tl).c_str());
            for (int i = 0; i < NR(); ++i) mul(i, d0, true);
            o("}\n");
        }
        return;
    }
    if (unit_code(d0) == 0 && unit_code(d1) < 0 && !(t_pend && t_pend[tpos])) {
        if (!((t_pdm >> tpos) & 1)) t_pd[tpos] = make_double2(1.0, 0.0);
        t_pd[tpos] = cmulh(t_pd[tpos], d1);  // pending on slot tpos's hi half
        t_pdm |= 1u << tpos;
        return;
    }
    pd_flush(o, tpos);
    for (int i = 0; i < NR(); ++i) mul(i, ((i >> tpos) & 1) ? d1 : d0, false);
}

// apply slot s's pending constant to its hi half
void pd_flush(Out &o, int s) {
    if (!((t_pdm >> s) & 1) || !t_code) return;
    const double2 d = t_pd[s];
    for (int i = 0; i < NR(); ++i) {
        if (!((i >> s) & 1)) continue;
        o("{ const d2 X = v[%d]; v[%d] = %s; }\n", i, i, cm_fold(d, t_code[i]).c_str());
        t_code[i] = 0;
    }
    t_pdm &= ~(1u << s);
}

// register i's product of pending slot constants (1 if none)
double2 pd_of(int i) {
    double2 c = make_double2(1.0, 0.0);
    for (int s = 0; s < NS(); ++s)
        if (((t_pdm >> s) & 1) && ((i >> s) & 1)) c = cmulh(c, t_pd[s]);
    return c;
}

}  // namespace

bool pend_on() { return true; }

// Tile pipelining modes of the generated kernel:
//   0  one shared buffer, 4 CTAs/SM; the first group reads HBM directly when
//      its rows are coalesced, otherwise cp.async fills the buffer first
//   1  two shared buffers, 3 CTAs/SM: tile i+1 streams in (cp.async) while
//      the groups of tile i run; the first group reads shared memory
//   2  one buffer, 4 CTAs/SM: once the last group has read its registers the
//      buffer is free, so the next tile's cp.async fill is issued there and
//      overlaps the last group's arithmetic and direct HBM stores (passes
//      without a direct last group use mode 0)
//   3  tile ring (12-qubit tiles with a direct last group; measured, not
//      the default): one CTA per SM of two warpgroups, each running the pass's
//      groups on its own tiles (even / odd tile numbers of the CTA), three
//      64 KiB buffers shared round-robin (tile j in buffer j % 3).  The
//      warpgroup that has read its last group out of a buffer refills it
//      at once with tile j + 3 -- the OTHER warpgroup's next-but-one tile
//      -- so a fill has about half a tile period of lead instead of only the
//      last group's arithmetic; an mbarrier per buffer (cp.async arrivals)
//      tells the consumer when its tile has landed.  Transitions sync the
//      warpgroup only (named barriers).  ncu of mode 2 on configs[1]: 24 % of
//      the warps' stall samples sat at the tile-start fill wait; the ring
//      cut that to ~5 % but ran configs[1] 4 % slower (DRAM throughput of
//      light passes fell, STG / LDS queue stalls rose: 117.0k vs 121-123k).
//   4  split prefetch (12-qubit tiles with a direct last group; measured, not
//      the default -- configs[1] 123.9k vs mode 2's 123.5k, within noise):
//      mode 2's two CTAs per SM, each with its 64 KiB working buffer W plus
//      a 32 KiB buffer F.  A tile is filled in halves: half A (the fill's
//      registers 0-15, byte offsets < 32 KiB) into F as soon as the first
//      group of the previous tile has read F -- a whole tile of lead -- and
//      half B (offsets >= 32 KiB) into its own place in W once the last
//      group has its registers, as in mode 2 but half the bytes.  The first
//      group reads through the affine map o -> o + 64 KiB * (o < 32 KiB).
int jit_mode() {
    static int m = [] {
        const char *e = getenv("SVB_JIT_MODE");
        int v = e ? atoi(e) : -1;
        return (v >= 0 && v <= 4) ? v : -1;
    }();
    return m;
}

// default per tile size: fm 11 runs 4 CTAs/SM, which already overlap one
// another's loads; fm 12/13 run 2 / 1 CTAs per SM and need the prefetch
// (measured on configs[1]: fm 13 mode 0 75.2k, mode 2 86.6k gate apps/s)
int jit_pass_mode(const FPass &P) {
    int m = jit_mode();
    if (m < 0) m = P.fm > 11 ? 2 : 0;
    if (m == 1 && P.fm != 11) m = 0;  // two tiles fit only at fm 11
    if ((m == 3 || m == 4) && (P.fm != 12 || P.fs < 5)) m = 2;  // 64 KiB tiles, 32 registers per thread
    if ((m == 2 || m == 3 || m == 4) && !P.direct_last) m = 0;
    return m;
}

// threads of one tile's worker (a warpgroup in mode 3)
static int jit_wg_threads(const FPass &P) { return (1 << P.fm) >> P.fs; }

int jit_threads(const FPass &P) { return (jit_pass_mode(P) == 3 ? 2 : 1) * jit_wg_threads(P); }

// resident CTAs per SM the generated kernel is built for (__launch_bounds__):
// 64K registers / (threads x registers per thread)
int jit_ctas_per_sm(const FPass &P) {
    if (jit_pass_mode(P) == 1) return 3;
    if (jit_pass_mode(P) == 3) return 1;
    // 16 amplitudes per thread fit 128 registers, 32 need the full 255
    return std::max(1, 65536 / (jit_threads(P) * (P.fs >= 5 ? 256 : 128)));
}
// tile buffers live in dynamic shared memory when they exceed the 48 KiB
// static limit (double buffering, or tiles of 12+ qubits)
size_t jit_dyn_smem(const FPass &P) {
    const int m = jit_pass_mode(P);
    const size_t t = (size_t(1) << P.fm) * sizeof(double2);
    const size_t b = m == 1 ? 2 * t : m == 3 ? 3 * t : m == 4 ? t + t / 2 : t;
    return b > 40 * 1024 ? b : 0;
}


// Thread-index copy the compiler cannot see through: per-thread address
// terms are recomputed where they are used instead of being hoisted out of
// the tile loop and kept live (or spilled) across the gate arithmetic.
const char *kOpaqueTid = "unsigned tg = tid; asm volatile(\"\" : \"+r\"(tg));\n";

// SVB_JIT_RESWZ=0 keeps the planner's swizzles (measurement)
bool t_reswz_on() {
    static const bool on = [] {
        const char *e = getenv("SVB_JIT_RESWZ");
        return !e || atoi(e) != 0;
    }();
    return on;
}

// Re-search the swizzle of the transition A -> B (fused.cu, "Shared-memory
// swizzle per transition": an XOR-linear map h of a local index's bits >= 3
// into its 16 B chunk number) when A's pending swaps `pend` make its store
// phases conflict: lane bit j of the store carries A's thread term j plus the
// slot term of every pending swap whose condition contains thread bit j.
void reswizzle(FGroup &A, FGroup &B, const uint64_t *pend, int fm, int tbits) {
    const int fs = NS();
    auto ways3 = [](int a, int b, int c) {
        int seen[8] = {0}, w = 0;
        for (int l = 0; l < 8; ++l) w = std::max(w, ++seen[((l & 1) ? a : 0) ^ ((l & 2) ? b : 0) ^ ((l & 4) ? c : 0)]);
        return w;
    };
    auto chunk = [](uint32_t off) { return int(off >> 4) & 7; };
    bool lane_pend = false;
    int eff[3];
    for (int j = 0; j < 3; ++j) {
        eff[j] = chunk(A.st_t[j]);
        for (int k = 0; k < fs; ++k)
            if ((pend[k] >> j) & 1) {
                eff[j] ^= chunk(A.st_s[k]);
                lane_pend = true;
            }
    }
    if (!lane_pend || ways3(eff[0], eff[1], eff[2]) <= 1) return;
    typedef std::array<int, FMMAX> Hmap;
    auto bank = [&](int v, const Hmap &h) {
        int c = v & 7;
        for (int j = 3; j < fm; ++j)
            if ((v >> j) & 1) c ^= h[j];
        return c;
    };
    auto cost = [&](const Hmap &h) {
        int e[3];
        for (int j = 0; j < 3; ++j) {
            e[j] = bank(A.mcol[A.tmap[j]], h);
            for (int k = 0; k < fs; ++k)
                if ((pend[k] >> j) & 1) e[j] ^= bank(A.mcol[A.pos[k]], h);
        }
        return ways3(e[0], e[1], e[2]) +
               ways3(bank(B.qcol[B.tmap[0]], h), bank(B.qcol[B.tmap[1]], h), bank(B.qcol[B.tmap[2]], h));
    };
    Hmap best{};
    int bc = 1 << 30;
    uint32_t rng = 0x2545f491u;
    for (int tries = 0; tries < 2000 && bc > 2; ++tries) {
        Hmap h{};
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
    // the swizzle in force costs ways(eff) + 1 at best; keep it unless the search found better
    if (bc >= ways3(eff[0], eff[1], eff[2]) + 1) return;
    auto off = [&](int v) { return (uint32_t)(16 * ((v & ~7) | bank(v, best))); };
    for (int j = 0; j < tbits; ++j) {
        A.st_t[j] = off(A.mcol[A.tmap[j]]);
        B.ld_t[j] = off(B.qcol[B.tmap[j]]);
    }
    for (int k = 0; k < fs; ++k) {
        A.st_s[k] = off(A.mcol[A.pos[k]]);
        B.ld_s[k] = off(B.qcol[B.pos[k]]);
    }
    A.st_b = off(A.mb);
    B.ld_b = off(B.qb);
}

// Overlap between a group's shared-memory stores and other threads' loads
// of the same group: 0 none (each thread rewrites only chunks it read), 1
// within warps only, 2 across warps.  Pending swaps only exchange a thread's
// own store slots, so the per-thread store set is the one computed here.
int store_hazard(const FGroup &G, int threads, int tbits) {
    const int nr = NR();
    std::unordered_map<unsigned, int> owner;
    owner.reserve(size_t(threads) * nr);
    for (int t = 0; t < threads; ++t) {
        unsigned a = G.ld_b;
        for (int j = 0; j < tbits; ++j)
            if ((t >> j) & 1) a ^= G.ld_t[j];
        for (int r = 0; r < nr; ++r) owner[a ^ xcombo_h(G.ld_s, r)] = t;
    }
    int hz = 0;
    for (int t = 0; t < threads && hz < 2; ++t) {
        unsigned b = G.st_b;
        for (int j = 0; j < tbits; ++j)
            if ((t >> j) & 1) b ^= G.st_t[j];
        for (int r = 0; r < nr; ++r) {
            auto it = owner.find(b ^ xcombo_h(G.st_s, r));
            if (it == owner.end() || it->second == t) continue;
            hz = std::max(hz, it->second / 32 == t / 32 ? 1 : 2);
        }
    }
    return hz;
}

// variant: 0 exact, 1 FMA, 2 FMA + factor extraction (F: the global factor
// carried in and out; last: the circuit's last fused pass, which applies F)
std::string jit_body(const FPass &P, int variant, double2 &F, bool last);

std::string jit_source(const FPass &P, int variant, double2 &F, bool last) {
    ConstPool pool;
    t_pool = &pool;
    t_fs = P.fs;
    std::string body = jit_body(P, variant, F, last);
    t_pool = nullptr;
    Out o;
    o("#define SVB_FMA %d\n", variant >= 1 ? 1 : 0);
    o.s += kPreamble;
    o("__constant__ double kc[%d] = {", std::max<int>(1, (int)pool.vals.size()));
    for (size_t i = 0; i < pool.vals.size(); ++i) o("%s%s", i ? ", " : "", hexf(pool.vals[i]).c_str());
    if (pool.vals.empty()) o("0.0");
    o("};\n");
    return o.s + body;
}

std::string jit_body(const FPass &P, int variant, double2 &F, bool last) {
    const bool fma = variant >= 1, fast = variant == 2;
    const int mode = jit_pass_mode(P);
    Out o;
    const int FTILE = 1 << P.fm, FTHREADS = jit_wg_threads(P), FTBITS = P.fm - P.fs;
    const bool ring = mode == 3;
    const bool split = mode == 4;
    // CTA-wide barrier, or the warpgroup's own in the ring
    const std::string SYNC = ring ? "wg_sync(wg, " + std::to_string(FTHREADS) + ");" : "__syncthreads();";
    const int colmask = (1 << P.flow) - 1;
    // Tile-local global offsets are XOR-linear in the thread index and the
    // register number: thread parts are computed per use from the opaque
    // index, register parts are constants.  They fit 32 bits while every
    // tile qubit is < 32 (always, for one GPU's <= 2^31-amplitude slab), so
    // an address is one XOR plus one IMAD.WIDE off the tile pointer pa.
    int maxbit = P.flow - 1;
    for (int j = 0; j < P.fm - P.flow; ++j) maxbit = std::max(maxbit, (int)P.rowbit[j]);
    const bool narrow = maxbit < 32;
    const char *OFF = narrow ? "unsigned" : "i64";
    auto offl = [&](int64_t v) {
        char b[40];
        if (narrow)
            snprintf(b, sizeof b, "%uu", (unsigned)v);
        else
            snprintf(b, sizeof b, "%lldll", (long long)v);
        return std::string(b);
    };
    int lt = 0;  // log2(threads)
    while ((1 << lt) < FTHREADS) ++lt;
    // element e = tid + k * threads: column = tid's low flow bits, row bits =
    // tid's remaining bits then k's bits
    auto row_off = [&](int rbit) { return int64_t(1) << P.rowbit[rbit]; };
    o("extern \"C\" __global__ void __launch_bounds__(%d, %d) kpass(d2 *__restrict__ a, i64 ntiles) {\n",
      jit_threads(P), jit_ctas_per_sm(P));
    if (jit_dyn_smem(P))
        o("extern __shared__ d2 dsm[];\n");
    else
        o("__shared__ alignas(16) d2 dsm[%d];\n", FTILE);
    if (ring) {
        o("__shared__ unsigned long long mbar[3];\n");
        o("const int wg = threadIdx.x >> %d;\n", [&] { int l = 0; while ((1 << l) < FTHREADS) ++l; return l; }());
        o("const int tid = threadIdx.x & %d;\n", FTHREADS - 1);
    } else {
        o("const int tid = threadIdx.x;\n");
    }
    o("auto tbase = [&](i64 t) { i64 b = 0;\n");
    for (int j = 0; j < P.ncomp; ++j) o("b |= ((t >> %d) & 1) << %d;\n", j, P.comp[j]);
    o("return b; };\n");
    // per-thread (global row/column offset, swizzled smem byte offset) of element tid
    auto thread_parts = [&]() {
        o("%s r = tg & %d; unsigned s = 0;\n", OFF, colmask);
        for (int j = 0; j < lt; ++j) {
            if (j >= P.flow) o("if ((tg >> %d) & 1) r ^= %s;\n", j, offl(row_off(j - P.flow)).c_str());
            o("if ((tg >> %d) & 1) s ^= %uu;\n", j, (unsigned)(16 * swz_h(1 << j)));
        }
    };
    auto k_row = [&](int k) {
        int64_t v = 0;
        for (int b = 0; (1 << b) <= k; ++b)
            if ((k >> b) & 1) v ^= row_off(lt - P.flow + b);
        return v;
    };
    auto k_smem = [&](int k) { return (unsigned)(16 * swz_h(k * FTHREADS)); };
    // Global addresses as base + constant.  The thread's offset r and a
    // register's offset k_row(k) are XORs of different address bits, so
    // r ^ k_row(k) == r + k_row(k): one 64-bit pointer per thread and the
    // register part as the access's immediate offset (a per-access XOR costs
    // five integer instructions of 64-bit address arithmetic; the heaviest
    // configs[1] passes, whose bodies overflow the instruction cache, ran 13 %
    // faster without them).
    bool fill_add = true;
    {
        int64_t tm = colmask;
        for (int j = P.flow; j < lt; ++j) tm |= row_off(j - P.flow);
        for (int k = 0; k < NR(); ++k)
            if (k_row(k) & tm) fill_add = false;
    }
    auto fill_ptr = [&]() { if (fill_add) o("const d2 *const pr = p + r;\n"); };
    auto fill_src = [&](int k) {
        return fill_add ? "pr + " + offl(k_row(k)) : "p + (r ^ " + offl(k_row(k)) + ")";
    };
    if (ring) {
        // buffer byte offset bo (a multiple of 2^16) XORed into the shared
        // address, which stays a 32-bit shared-window offset
        o("const unsigned sbase = su32(dsm);\n");
        o("auto fill = [&](unsigned bo, const d2 *p) {\n%s", kOpaqueTid);
        thread_parts();
        o("s ^= bo;\n");
        fill_ptr();
        for (int k = 0; k < NR(); ++k)
            o("cpa_u(sbase + (s ^ %uu), %s);\n", k_smem(k), fill_src(k).c_str());
    } else {
        o("auto fill = [&](unsigned char *dstb, const d2 *p) {\n%s", kOpaqueTid);
        thread_parts();
        fill_ptr();
        for (int k = 0; k < NR(); ++k)
            o("cpa(dstb + (s ^ %uu), %s);\n", k_smem(k), fill_src(k).c_str());
    }
    if (ring)
        o("};\n(void)fill;\n");
    else
        o("asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\"); };\n(void)fill;\n");
    if (split) {
        // the fill's registers 0..NR/2-1 are the tile's bytes [0, 32K) (the
        // top register bit is element bit fm-1, byte bit 15): half A goes to
        // F = [64K, 96K), half B to its own place in W = [32K, 64K)
        for (int h = 0; h < 2; ++h) {
            o("auto fill%c = [&](const d2 *p) {\n%s", h ? 'B' : 'A', kOpaqueTid);
            thread_parts();
            fill_ptr();
            for (int k = h * NR() / 2; k < (h + 1) * NR() / 2; ++k)
                o("cpa(reinterpret_cast<unsigned char *>(dsm) + (s ^ %uu), %s);\n",
                  k_smem(k) + (h ? 0u : 0x10000u), fill_src(k).c_str());
            o("asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\"); };\n");
        }
    }
    // Direct HBM loads / stores of a group: address = pa + (x0 ^ combo(i)), x0
    // the thread's XOR-linear offset, combo(i) the XOR of the slot terms of
    // register i.  A slot term that shares no bit with any thread-varying
    // term, the constant start or another slot term only ever adds to the
    // address: those go into the access as a constant offset off a per-thread
    // pointer; the others (a CNOT folded into the map, a pending swap) keep
    // the XOR, one pointer per pattern of them.
    auto direct_access = [&](const char *x0, int64_t b, const int64_t *t, const int64_t *sl, const uint64_t *pend,
                             const std::function<void(int, const std::string &)> &emit) {
        int64_t vary = b;
        for (int j = 0; j < FTBITS; ++j) vary |= t[j];
        for (int k = 0; k < NS(); ++k)
            if (pend && pend[k]) vary |= sl[k];
        unsigned xset = 0;  // slot bits that keep the XOR
        for (int k = 0; k < NS(); ++k) {
            int64_t others = vary;
            for (int k2 = 0; k2 < NS(); ++k2)
                if (k2 != k) others |= sl[k2];
            if ((sl[k] & others) || (pend && pend[k])) xset |= 1u << k;
        }
        if (__builtin_popcount(xset) > 2) xset = (1u << NS()) - 1;  // too many pointers: plain XOR form
        const bool all_xor = xset == (1u << NS()) - 1;
        if (!all_xor)
            for (int i = 0; i < NR(); ++i) {
                if (unsigned(i) & ~xset) continue;  // i is a pattern of XOR slots only
                o("d2 *const p%s_%d = pa + (%s ^ %s);\n", x0, i, x0, offl(xcombo_g(sl, i)).c_str());
            }
        for (int i = 0; i < NR(); ++i) {
            if (all_xor) {
                emit(i, std::string("pa + (") + x0 + " ^ " + offl(xcombo_g(sl, i)) + ")");
            } else {
                emit(i, std::string("p") + x0 + "_" + std::to_string(unsigned(i) & xset) + " + " + offl(xcombo_g(sl, unsigned(i) & ~xset)));
            }
        }
    };
    const char *wait_all = "asm volatile(\"cp.async.wait_group 0;\\n\" ::: \"memory\");\n";
    const bool direct_first = P.direct_first && mode == 0;
    if (ring) {
        // tile j of this CTA = blockIdx.x + j * gridDim.x, buffer j % 3,
        // worked by warpgroup j & 1; its fill completes mbar[j % 3]'s phase j / 3
        o("auto fill3 = [&](int bi, i64 j) {\n"
          "const i64 t = blockIdx.x + j * gridDim.x;\n"
          "if (t < ntiles) { fill((unsigned)bi << 16, a + tbase(t)); mb_arrive_cp(&mbar[bi]); } };\n");
        o("if (threadIdx.x < 3) mb_init(&mbar[threadIdx.x], %d);\n__syncthreads();\n", FTHREADS);
        o("if (wg == 0) { fill3(0, 0); fill3(2, 2); } else { fill3(1, 1); }\n");
        o("for (i64 j = wg;; j += 2) {\n"
          "const i64 tix = blockIdx.x + j * gridDim.x;\n"
          "if (tix >= ntiles) break;\n"
          "const int bi = (int)(j %% 3);\n");
        o("d2 *const pa = a + tbase(tix);\n");
        o("d2 *buf = dsm + bi * %d;\n", FTILE);
        o("mb_wait(&mbar[bi], (unsigned)((j / 3) & 1));\n");
    } else {
        if (split)
            o("if (blockIdx.x < ntiles) { fillA(a + tbase(blockIdx.x)); fillB(a + tbase(blockIdx.x)); }\n");
        else if (mode != 0)
            o("if (blockIdx.x < ntiles) fill(reinterpret_cast<unsigned char *>(dsm), a + tbase(blockIdx.x));\n");
        o("int it = 0;\nfor (i64 tix = blockIdx.x; tix < ntiles; tix += gridDim.x, ++it) {\n");
        o("d2 *const pa = a + tbase(tix);\n");
    }
    if (ring) {
    } else if (mode == 1) {
        o("d2 *buf = dsm + (it & 1) * %d;\n", FTILE);
        o.s += wait_all;
        o("__syncthreads();\n{ const i64 nx = tix + gridDim.x; if (nx < ntiles) "
          "fill(reinterpret_cast<unsigned char *>(dsm + ((it + 1) & 1) * %d), a + tbase(nx)); }\n",
          FTILE);
    } else {
        o("d2 *buf = dsm;\n");
        if (mode == 2 || split) {
            o.s += wait_all;
            o("__syncthreads();\n");
        } else if (!direct_first) {
            o("fill(reinterpret_cast<unsigned char *>(buf), pa);\n");
            o.s += wait_all;
            o("__syncthreads();\n");
        }
    }
    if (ring) {
        // buffer bi starts at byte bi << 16 of the tile area and every in-tile
        // byte offset is < 2^16: the buffer folds into the per-thread XOR base
        // (bo), so shared accesses keep the constant dsm base and the XOR
        // address form (no per-access add)
        o("unsigned char *sb = reinterpret_cast<unsigned char *>(dsm);\n(void)buf;\n");
        o("const unsigned bo = (unsigned)bi << 16;\n");
    } else {
        o("unsigned char *sb = reinterpret_cast<unsigned char *>(buf);\n");
    }
    o("d2 v[%d];\n", NR());
    // (the groups' shared-memory maps may be re-swizzled below: a local copy)
    std::vector<FGroup> GR(P.groups, P.groups + P.ngroups);
    for (int gi = 0; gi < P.ngroups; ++gi) {
        FGroup Gx;
        if (split && gi == 0) {
            // first group: bytes [0, 32K) of the tile sit in F at +64K.  The
            // map o -> o ^ L(o) ^ K (L: byte bit 15 -> bit 16, K = 64K) is
            // affine, so every XOR term c becomes c ^ L(c), the base also ^ K
            Gx = GR[0];
            auto L = [](uint32_t c) { return c ^ (((c >> 15) & 1u) << 16); };
            Gx.ld_b = L(Gx.ld_b) ^ 0x10000u;
            for (int j = 0; j < FTBMAX; ++j) Gx.ld_t[j] = L(Gx.ld_t[j]);
            for (int k = 0; k < FSMAX; ++k) Gx.ld_s[k] = L(Gx.ld_s[k]);
        }
        const FGroup &G = (split && gi == 0) ? Gx : GR[gi];
        const bool last_group = gi == P.ngroups - 1;
        o("{ // group %d\n", gi);
        if (gi == 0 && direct_first) {
            o("%s g0 = %s;\n", OFF, offl(P.gl_b).c_str());
            o.s += kOpaqueTid;
            for (int j = 0; j < FTBITS; ++j) o("if ((tg >> %d) & 1) g0 ^= %s;\n", j, offl(P.gl_t[j]).c_str());
            direct_access("g0", P.gl_b, P.gl_t, P.gl_s, nullptr, [&](int i, const std::string &adr) {
                o("v[%d] = ldcs(%s);\n", i, adr.c_str());
            });
        } else {
            o("unsigned a0 = %uu%s;\n", (unsigned)G.ld_b, ring ? " ^ bo" : "");
            o.s += kOpaqueTid;
            for (int j = 0; j < FTBITS; ++j) o("if ((tg >> %d) & 1) a0 ^= %uu;\n", j, (unsigned)G.ld_t[j]);
            for (int i = 0; i < NR(); ++i)
                o("v[%d] = *reinterpret_cast<const d2 *>(sb + (a0 ^ %uu));\n", i, xcombo_h(G.ld_s, i));
        }
        if (last_group && mode == 2) {
            // every thread has its registers: refill the buffer with the next tile
            o("__syncthreads();\n{ const i64 nx = tix + gridDim.x; if (nx < ntiles) "
              "fill(reinterpret_cast<unsigned char *>(dsm), a + tbase(nx)); }\n");
        }
        if (last_group && split) {
            // registers in hand: W's half B (and, when this is also the first
            // group, F) take the next tile
            o("__syncthreads();\n{ const i64 nx = tix + gridDim.x; if (nx < ntiles) { %sfillB(a + tbase(nx)); } }\n",
              gi == 0 ? "fillA(a + tbase(nx)); " : "");
        }
        if (last_group && ring) {
            // the warpgroup has its registers: the buffer takes tile j + 3
            o("%s\nfill3(bi, j + 3);\n", SYNC.c_str());
        }
        uint64_t pend[FSMAX] = {0};
        if (fma && pend_on()) t_pend = pend;
        if (fast) {
            int code[FREGMAX] = {0};
            t_code = code;
            t_phase = false;
            t_phase_sign = false;
            t_hs = 0;
            t_pdm = 0;
            o("d2 ph = mk(1.0, 0.0);\n");
            for (int k = 0; k < NS(); ++k) o("d2 hs%d = mk(1.0, 0.0);\n", k);
            std::vector<TilePhase> tph;
            std::vector<SlotTilePhase> shs[FSMAX];
            t_tph = &tph;
            t_shs = shs;
            for (int q = G.first; q < G.first + G.count; ++q) emit_gate_fast(o, P.gates[q], code, F);
            flush_tile_phases(o);  // (ph is only read below, at the group's end)
            for (int k = 0; k < NS(); ++k) materialize_slot_tile(o, k);  // (hs<k> too)
            t_tph = nullptr;
            t_shs = nullptr;
            const double mag = cabsh(F);
            const bool applyF = gi == P.ngroups - 1 && (last || mag < 0x1p-200 || mag > 0x1p200) &&
                                !(F.x == 1.0 && F.y == 0.0);
            if (!t_phase && !applyF)  // nothing multiplies every register: per-slot phases alone
                for (int k = 0; k < NS(); ++k) slot_phase_flush(o, k);
            if (t_phase && t_phase_sign && !applyF && !t_pdm && !t_hs) {
                // ph is +-1: flip the sign bits of every register (integer pipe)
                // instead of a complex multiply; pending unit factors commute
                o("{ const unsigned pm = (unsigned)__double2hiint(ph.x) & 0x80000000u;\n");
                for (int i = 0; i < NR(); ++i) o("v[%d] = mk(cneg(v[%d].x, pm), cneg(v[%d].y, pm));\n", i, i, i);
                o("}\n");
            } else if (t_phase || applyF) {
                // every register is multiplied anyway (ph and / or F): the
                // pending per-slot phases hs (runtime) and constants (pd) ride
                // on that multiply -- one per-thread scalar per pattern of
                // pending slots a register lies in, one multiply per register
                const bool rt = t_phase;  // runtime base (ph) or compile-time (F)
                if (rt && applyF) {
                    o("ph = cm(%s, %s, ph);\n", lit(F.x).c_str(), lit(F.y).c_str());
                    F = make_double2(1.0, 0.0);
                }
                std::vector<unsigned> made;  // patterns whose scalar exists
                for (int i = 0; i < NR(); ++i) {
                    const unsigned hpat = t_hs & unsigned(i), ppat = t_pdm & unsigned(i);
                    const double2 c = rt ? pd_of(i) : cmulh(F, pd_of(i));
                    if (!rt && !hpat) {  // a compile-time constant
                        o("{ const d2 X = v[%d]; v[%d] = %s; }\n", i, i, cm_fold(c, code[i]).c_str());
                        code[i] = 0;
                        continue;
                    }
                    std::string var = "ph";
                    if (hpat || ppat || !rt) {
                        const unsigned key = hpat | (ppat << NS());
                        var = "fm" + std::to_string(key);
                        if (std::find(made.begin(), made.end(), key) == made.end()) {
                            made.push_back(key);
                            // base (ph, or the constant F * pd), times hs of the
                            // register's pending slots, times the constant pd
                            const std::string acc = rt ? "ph" : "mk(" + lit(c.x) + ", " + lit(c.y) + ")";
                            o("d2 %s = %s;\n", var.c_str(), acc.c_str());
                            for (int k = 0; k < NS(); ++k)
                                if ((hpat >> k) & 1) o("%s = cm(hs%d.x, hs%d.y, %s);\n", var.c_str(), k, k, var.c_str());
                            if (rt && ppat)
                                o("%s = cm(%s, %s, %s);\n", var.c_str(), lit(c.x).c_str(), lit(c.y).c_str(),
                                  var.c_str());
                        }
                    }
                    std::string e = cm_ph(code[i]);
                    for (size_t at; (at = e.find("ph.")) != std::string::npos;) e.replace(at, 3, var + "#");
                    for (size_t at; (at = e.find("#")) != std::string::npos;) e.replace(at, 1, ".");
                    o("{ const d2 X = v[%d]; v[%d] = %s; }\n", i, i, e.c_str());
                    code[i] = 0;
                }
                for (int k = 0; k < NS(); ++k)
                    if ((t_hs >> k) & 1) o("hs%d = mk(1.0, 0.0);\n", k);
                t_hs = 0;
                t_pdm = 0;
                if (applyF) F = make_double2(1.0, 0.0);
            } else if (t_pdm) {  // the pending slot constants alone, one multiply per register
                for (int i = 0; i < NR(); ++i) {
                    if (!(t_pdm & unsigned(i))) continue;
                    o("{ const d2 X = v[%d]; v[%d] = %s; }\n", i, i, cm_fold(pd_of(i), code[i]).c_str());
                    code[i] = 0;
                }
                t_pdm = 0;
            }
            for (int i = 0; i < NR(); ++i) materialize(o, code, i);
        } else if (fma) {
            int code[FREGMAX] = {0};
            t_code = code;
            for (int q = G.first; q < G.first + G.count; ++q) emit_gate_fold(o, P.gates[q], code);
            for (int i = 0; i < NR(); ++i) materialize(o, code, i);
        } else {
            for (int q = G.first; q < G.first + G.count; ++q) emit_gate(o, P.gates[q]);
        }
        t_pend = nullptr;
        t_code = nullptr;
        if (last_group && P.direct_last) {
            if (G.perm && gi == 0 && direct_first) o("%s\n", SYNC.c_str());
            o("%s s0 = %s;\n", OFF, offl(P.gs_b).c_str());
            o("{\n%s", kOpaqueTid);
            for (int j = 0; j < FTBITS; ++j) o("if ((tg >> %d) & 1) s0 ^= %s;\n", j, offl(P.gs_t[j]).c_str());
            for (int k = 0; k < NS(); ++k)  // pending swaps: per-thread store address
                if (pend[k]) o("if (%s) s0 ^= %s;\n", pcond(pend[k]).c_str(), offl(P.gs_s[k]).c_str());
            o("}\n");
            direct_access("s0", P.gs_b, P.gs_t, P.gs_s, pend, [&](int i, const std::string &adr) {
                o("stcs(%s, v[%d]);\n", adr.c_str(), i);
            });
        } else {
            // the store overwrites chunks other threads may not have loaded
            // yet (the swizzle changes per transition): order them with the
            // narrowest barrier that covers every overlap
            // A pending swap conditioned on lane bits 0-2 XORs its slot's
            // store term into some lanes' addresses, chunk bits included: the
            // 8-lane phases the planner made conflict-free (it cannot know
            // the pending swaps) may then hit a bank group twice.  configs[1]:
            // 63 of 355 store phases ran 2-way conflicts (ncu: every STS of
            // such a phase at twice its wavefronts).  Search this
            // transition's swizzle again with the lanes' real XOR terms and
            // move this group's store map and the next group's load map to it.
            if (t_reswz_on() && !(split && gi == 0)) reswizzle(GR[gi], GR[gi + 1], pend, P.fm, FTBITS);
            const int hz = (gi == 0 && direct_first) ? 0 : store_hazard(G, FTHREADS, FTBITS);
            if (G.perm)
                o("%s\n", SYNC.c_str());
            else if (hz == 2)
                o("%s  // cross-warp store hazard\n", SYNC.c_str());
            else if (hz == 1)
                o("__syncwarp();\n");
            o("unsigned b0 = %uu%s;\n", (unsigned)G.st_b, ring ? " ^ bo" : "");
            o("{\n%s", kOpaqueTid);
            for (int j = 0; j < FTBITS; ++j) o("if ((tg >> %d) & 1) b0 ^= %uu;\n", j, (unsigned)G.st_t[j]);
            for (int k = 0; k < NS(); ++k)
                if (pend[k]) o("if (%s) b0 ^= %uu;\n", pcond(pend[k]).c_str(), (unsigned)G.st_s[k]);
            o("}\n");
            for (int i = 0; i < NR(); ++i)
                o("*reinterpret_cast<d2 *>(sb + (b0 ^ %uu)) = v[%d];\n", xcombo_h(G.st_s, i), i);
            o("%s\n", SYNC.c_str());
            if (split && gi == 0)  // every thread has read F: it takes the next tile's half A
                o("{ const i64 nx = tix + gridDim.x; if (nx < ntiles) fillA(a + tbase(nx)); }\n");
        }
        o("}\n");
    }
    if (!P.direct_last) {
        o("{\n%s", kOpaqueTid);
        thread_parts();
        if (fill_add) o("d2 *const pw = pa + r;\n");
        for (int k = 0; k < NR(); ++k)
            if (fill_add)
                o("pw[%s] = *reinterpret_cast<const d2 *>(sb + (s ^ %uu));\n", offl(k_row(k)).c_str(), k_smem(k));
            else
                o("pa[r ^ %s] = *reinterpret_cast<const d2 *>(sb + (s ^ %uu));\n", offl(k_row(k)).c_str(), k_smem(k));
        o("}\n");
    }
    // mode 0: the buffer must be free before the next tile's loads; modes 1/2
    // order reuse with the barrier after the next wait
    if (mode == 0) o("__syncthreads();\n");
    o("}\n");
    if (mode != 0 && !ring) o.s += wait_all;
    o("}\n");
    return o.s;
}

// ---------------------------------------------------------------------------
// compile + cache

// A loaded pass module, shared by every compiled plan that uses its source
// (plans hold shared_ptrs; the cache only weak ones, so a module is unloaded
// once the last plan using it leaves the plan cache -- bounded memory for
// long-running processes that see many circuits).
struct JitModule {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
    // (the plan holding the last reference drains every device it launched on
    // before releasing it -- ~CompiledPlan in fused.cu -- so no queued launch
    // of this module is outstanding here)
    ~JitModule() {
        if (lib) cudaLibraryUnload(lib);  // (errors at process teardown are harmless)
    }
};

static std::mutex g_jit_mu;
static std::unordered_map<uint64_t, std::weak_ptr<JitModule>> g_jit_cache;
static std::string g_jit_err;

static uint64_t hash_str(const std::string &s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return h;
}

// NVRTC is loaded at run time (dlopen): the library must load on hosts
// without a CUDA toolkit, and JIT is an optional accelerator -- if NVRTC is
// missing, fused passes run on the k_fused interpreter.
struct Nvrtc {
    typedef int (*create_t)(void **, const char *, const char *, int, const char *const *, const char *const *);
    typedef int (*compile_t)(void *, int, const char *const *);
    typedef int (*size_t_)(void *, size_t *);
    typedef int (*get_t)(void *, char *);
    typedef int (*destroy_t)(void **);
    typedef int (*version_t)(int *, int *);
    create_t create = nullptr;
    compile_t compile = nullptr;
    size_t_ log_size = nullptr, cubin_size = nullptr;
    get_t log = nullptr, cubin = nullptr;
    destroy_t destroy = nullptr;
    int major = 0, minor = 0;
    bool ok = false;
};

static const Nvrtc &nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        const char *cands[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"};
        void *h = nullptr;
        for (const char *c : cands)
            if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return r;
        r.create = (Nvrtc::create_t)dlsym(h, "nvrtcCreateProgram");
        r.compile = (Nvrtc::compile_t)dlsym(h, "nvrtcCompileProgram");
        r.log_size = (Nvrtc::size_t_)dlsym(h, "nvrtcGetProgramLogSize");
        r.log = (Nvrtc::get_t)dlsym(h, "nvrtcGetProgramLog");
        r.cubin_size = (Nvrtc::size_t_)dlsym(h, "nvrtcGetCUBINSize");
        r.cubin = (Nvrtc::get_t)dlsym(h, "nvrtcGetCUBIN");
        r.destroy = (Nvrtc::destroy_t)dlsym(h, "nvrtcDestroyProgram");
        if (auto v = (Nvrtc::version_t)dlsym(h, "nvrtcVersion")) v(&r.major, &r.minor);
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        return r;
    }();
    return n;
}

bool jit_available() { return nvrtc().ok; }

static const std::vector<const char *> &nvrtc_opts() {
    // (function-local statics a background compile uses are never destroyed:
    // one may still run while static destruction proceeds at process exit)
    static const std::vector<const char *> &opts = *new std::vector<const char *>([] {
        std::vector<const char *> o = {"-arch=sm_100a", "-std=c++17", "-default-device", "-fmad=false"};
        if (getenv("SVB_JIT_LINEINFO")) o.push_back("-lineinfo");  // for ncu source pages
        return o;
    }());
    return opts;
}

static bool nvrtc_compile_now(const std::string &src, std::vector<char> &cubin, std::string &log) {
    const Nvrtc &nv = nvrtc();
    if (!nv.ok) {
        log = "NVRTC not available";
        return false;
    }
    void *prog = nullptr;
    if (nv.create(&prog, src.c_str(), "svb_pass.cu", 0, nullptr, nullptr) != 0) {
        log = "nvrtcCreateProgram failed";
        return false;
    }
    const std::vector<const char *> &opts = nvrtc_opts();
    if (nv.compile(prog, (int)opts.size(), opts.data()) != 0) {
        size_t n = 0;
        nv.log_size(prog, &n);
        log.assign(n, '\0');
        nv.log(prog, &log[0]);
        nv.destroy(&prog);
        return false;
    }
    size_t n = 0;
    nv.cubin_size(prog, &n);
    cubin.resize(n);
    nv.cubin(prog, cubin.data());
    nv.destroy(&prog);
    return true;
}

// On-disk cubin cache: a circuit compiled once is not recompiled by the next
// process.  Directory: SVB_JIT_CACHE ("0" or "" disables), else
// $XDG_CACHE_HOME/svb-jit, else $HOME/.cache/svb-jit.  Entry name = two
// independent 64-bit hashes of (source, options, NVRTC version); the file
// carries a magic and the source length and hash, re-checked on read, and is
// written to a temporary name and renamed (concurrent writers are harmless).
static const std::string &jit_cache_dir() {
    static const std::string &dir = *new std::string([] {
        std::string d;
        if (const char *e = getenv("SVB_JIT_CACHE")) {
            d = e;
            if (d == "0") d.clear();
        } else if (const char *x = getenv("XDG_CACHE_HOME")) {
            if (*x) d = std::string(x) + "/svb-jit";
        } else if (const char *h = getenv("HOME")) {
            if (*h) d = std::string(h) + "/.cache/svb-jit";
        }
        if (!d.empty()) {  // mkdir -p
            for (size_t i = 1; i <= d.size(); ++i)
                if (i == d.size() || d[i] == '/') mkdir(d.substr(0, i).c_str(), 0755);
            struct stat st;
            if (stat(d.c_str(), &st) != 0 || !S_ISDIR(st.st_mode)) d.clear();
        }
        return d;
    }());
    return dir;
}

static uint64_t fnv64(const void *p, size_t n, uint64_t h) {
    const unsigned char *b = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

struct CubinKey {
    uint64_t a, b;
};

static CubinKey cubin_key(const std::string &src) {
    std::string k = src;
    for (const char *o : nvrtc_opts()) (k += '\0') += o;
    k += "\0nvrtc " + std::to_string(nvrtc().major) + "." + std::to_string(nvrtc().minor);
    // second hash: different offset basis and the bytes fed in reverse
    std::string r(k.rbegin(), k.rend());
    return {fnv64(k.data(), k.size(), 1469598103934665603ull), fnv64(r.data(), r.size(), 0x9e3779b97f4a7c15ull)};
}

static const uint64_t kCubinMagic = 0x31304a4954425653ull;  // "SVBTIJ01"

static std::string cubin_path(const CubinKey &key) {
    char name[48];
    snprintf(name, sizeof name, "/%016llx%016llx.cubin", (unsigned long long)key.a, (unsigned long long)key.b);
    return jit_cache_dir() + name;
}

static bool cubin_load(const std::string &src, const CubinKey &key, std::vector<char> &cubin) {
    FILE *f = fopen(cubin_path(key).c_str(), "rb");
    if (!f) return false;
    uint64_t hdr[3] = {0, 0, 0};
    bool ok = fread(hdr, sizeof hdr, 1, f) == 1 && hdr[0] == kCubinMagic && hdr[1] == src.size() &&
              hdr[2] == fnv64(src.data(), src.size(), 14695981039346656037ull ^ 0x5a5a);
    if (ok) {
        fseek(f, 0, SEEK_END);
        long end = ftell(f);
        ok = end > long(sizeof hdr);
        if (ok) {
            cubin.resize(size_t(end) - sizeof hdr);
            fseek(f, long(sizeof hdr), SEEK_SET);
            ok = fread(cubin.data(), 1, cubin.size(), f) == cubin.size();
        }
    }
    fclose(f);
    return ok;
}

static void cubin_store(const std::string &src, const CubinKey &key, const std::vector<char> &cubin) {
    const std::string path = cubin_path(key);
    char tmp_sfx[64];
    snprintf(tmp_sfx, sizeof tmp_sfx, ".tmp.%d.%zx", (int)getpid(),
             std::hash<std::thread::id>()(std::this_thread::get_id()));
    const std::string tmp = path + tmp_sfx;
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    const uint64_t hdr[3] = {kCubinMagic, src.size(), fnv64(src.data(), src.size(), 14695981039346656037ull ^ 0x5a5a)};
    bool ok = fwrite(hdr, sizeof hdr, 1, f) == 1 && fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
    ok = (fclose(f) == 0) && ok;
    if (!ok || rename(tmp.c_str(), path.c_str()) != 0) unlink(tmp.c_str());
}

static std::atomic<long> g_disk_hits{0}, g_compiles{0};

// Background compiles (SVB_RUN_JIT_ASYNC).  Outstanding threads are joined
// before this file's statics (the module cache they fill) are destroyed:
// the joiner is defined after them, so it is destroyed first.
struct AsyncJoiner {
    struct Job {
        std::thread t;
        std::shared_ptr<std::atomic<bool>> done;
    };
    std::mutex mu;
    std::vector<Job> jobs;
    ~AsyncJoiner() {
        std::vector<Job> j;
        {
            std::lock_guard<std::mutex> lk(mu);
            j.swap(jobs);
        }
        for (auto &x : j)
            if (x.t.joinable()) x.t.join();
    }
};
static AsyncJoiner g_async;

void jit_async(std::function<void()> fn) {
    std::lock_guard<std::mutex> lk(g_async.mu);
    for (auto it = g_async.jobs.begin(); it != g_async.jobs.end();) {  // reap finished compiles
        if (it->done->load()) {
            it->t.join();
            it = g_async.jobs.erase(it);
        } else {
            ++it;
        }
    }
    auto done = std::make_shared<std::atomic<bool>>(false);
    g_async.jobs.push_back({std::thread([fn = std::move(fn), done] {
                                fn();
                                done->store(true);
                            }),
                            done});
}

// Block until every background compile started so far has finished.
extern "C" void svb_jit_wait(void) {
    std::vector<AsyncJoiner::Job> j;
    {
        std::lock_guard<std::mutex> lk(g_async.mu);
        j.swap(g_async.jobs);
    }
    for (auto &x : j)
        if (x.t.joinable()) x.t.join();
}

extern "C" void svb_jit_counters(long *disk_hits, long *compiles) {
    if (disk_hits) *disk_hits = g_disk_hits.load();
    if (compiles) *compiles = g_compiles.load();
}

static bool nvrtc_compile(const std::string &src, std::vector<char> &cubin, std::string &log) {
    const bool disk = !jit_cache_dir().empty();
    CubinKey key{0, 0};
    if (disk) {
        key = cubin_key(src);
        if (cubin_load(src, key, cubin)) {
            ++g_disk_hits;
            return true;
        }
    }
    if (!nvrtc_compile_now(src, cubin, log)) return false;
    ++g_compiles;
    if (disk) cubin_store(src, key, cubin);
    return true;
}

// The >48 KiB dynamic shared-memory opt-in is a per-device attribute of a
// library kernel: it is set for the device a launch runs on, the first time a
// (kernel, device) pair is seen -- a plan loaded while cuda:0 was current
// still launches on cuda:1.
static bool set_dyn_smem(cudaKernel_t fn, size_t bytes, int d) {
    return cudaKernelSetAttributeForDevice(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes, d) ==
           cudaSuccess;
}

static bool ensure_dyn_smem(cudaKernel_t fn, size_t bytes) {
    if (!bytes) return true;
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return false;
    static std::mutex &mu = *new std::mutex;
    static auto &done = *new std::unordered_map<const void *, uint64_t>;  // kernel -> devices with the attribute
    std::lock_guard<std::mutex> lk(mu);
    uint64_t &mask = done[(const void *)fn];
    const uint64_t bit = d < 64 ? uint64_t(1) << d : 0;
    if (bit && (mask & bit)) return true;
    if (!set_dyn_smem(fn, bytes, d)) return false;
    mask |= bit;
    return true;
}

// Compile (or fetch) one kernel per pass.  Returns false and leaves
// `fns` empty on any failure (the caller falls back to k_fused).
int jit_variant(bool fma) { return fma ? (jit_factor_on() ? 2 : 1) : 0; }

bool jit_build(const std::vector<FPass> &passes, int variant, std::vector<void *> &fns,
               std::vector<std::shared_ptr<void>> &keep) {
    fns.assign(passes.size(), nullptr);
    keep.assign(passes.size(), nullptr);
    std::vector<std::string> srcs(passes.size());
    std::vector<uint64_t> keys(passes.size());
    std::vector<size_t> todo;
    double2 F = make_double2(1.0, 0.0);
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        for (size_t i = 0; i < passes.size(); ++i) {
            srcs[i] = jit_source(passes[i], variant, F, i + 1 == passes.size());
            keys[i] = hash_str(srcs[i]);
            auto it = g_jit_cache.find(keys[i]);
            std::shared_ptr<JitModule> m = it != g_jit_cache.end() ? it->second.lock() : nullptr;
            if (m) {
                fns[i] = (void *)m->fn;
                keep[i] = m;
            } else {
                todo.push_back(i);
            }
        }
    }
    if (!todo.empty()) {
        cudaFree(nullptr);  // make sure the runtime's primary context is current
        std::vector<std::vector<char>> cubins(passes.size());
        std::atomic<size_t> next{0};
        std::atomic<bool> ok{true};
        unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
            pool.emplace_back([&] {
                for (size_t k; (k = next++) < todo.size();) {
                    std::string log;
                    if (!nvrtc_compile(srcs[todo[k]], cubins[todo[k]], log)) {
                        ok = false;
                        std::lock_guard<std::mutex> lk(g_jit_mu);
                        g_jit_err = log.substr(0, 2000);
                    }
                }
            });
        for (auto &t : pool) t.join();
        if (!ok) {
            fprintf(stderr, "svb jit: compile failed, using the interpreter:\n%s\n", g_jit_err.c_str());
            fns.clear();
            keep.clear();
            return false;
        }
        std::lock_guard<std::mutex> lk(g_jit_mu);
        for (size_t i : todo) {
            auto m = std::make_shared<JitModule>();
            if (cudaLibraryLoadData(&m->lib, cubins[i].data(), nullptr, nullptr, 0, nullptr, nullptr, 0) !=
                    cudaSuccess ||
                cudaLibraryGetKernel(&m->fn, m->lib, "kpass") != cudaSuccess) {
                cudaGetLastError();
                fns.clear();
                keep.clear();
                return false;
            }
            g_jit_cache[keys[i]] = m;
            fns[i] = (void *)m->fn;
            keep[i] = m;
        }
        if (g_jit_cache.size() > 4096)  // drop entries whose modules are gone
            for (auto it = g_jit_cache.begin(); it != g_jit_cache.end();)
                it = it->second.expired() ? g_jit_cache.erase(it) : std::next(it);
    }
    return true;
}

// Host-only check: generate and NVRTC-compile every pass (no device needed).
int jit_compile_only(const std::vector<FPass> &passes, int variant, std::string &err) {
    const char *dump = getenv("SVB_JIT_DUMP");  // directory: write pass sources and cubins
    int k = 0;
    double2 F = make_double2(1.0, 0.0);
    for (const FPass &P : passes) {
        std::vector<char> cubin;
        std::string src = jit_source(P, variant, F, k + 1 == (int)passes.size());
        if (!nvrtc_compile(src, cubin, err)) return -1;
        if (dump) {
            std::string base = std::string(dump) + "/pass" + std::to_string(k);
            if (FILE *f = fopen((base + ".cu").c_str(), "w")) {
                fwrite(src.data(), 1, src.size(), f);
                fclose(f);
            }
            if (FILE *f = fopen((base + ".cubin").c_str(), "wb")) {
                fwrite(cubin.data(), 1, cubin.size(), f);
                fclose(f);
            }
        }
        ++k;
    }
    return (int)passes.size();
}

bool jit_launch(void *fn, const FPass &P, double2 *a, int64_t ntiles, cudaStream_t s) {
    static int sms = [] {
        int d = 0, v = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        return v;
    }();
    const int grid = (int)std::min<int64_t>(ntiles, int64_t(sms) * jit_ctas_per_sm(P));
    if (!ensure_dyn_smem((cudaKernel_t)fn, jit_dyn_smem(P))) return false;
    long long nt = ntiles;
    void *args[] = {&a, &nt};
    return cudaLaunchKernel((const void *)fn, dim3(grid), dim3(jit_threads(P)), args, jit_dyn_smem(P), s) ==
           cudaSuccess;
}

}  // namespace svb
