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
// arithmetic (exact or FMA), so its results equal the interpreter's bit for
// bit.  NVRTC compiles all passes of a plan in parallel host threads; modules
// are cached in memory by source hash.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "fused_desc.h"

namespace svb {

namespace {

struct Out {
    std::string s;
    void operator()(const char *fmt, ...) {
        char tmp[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(tmp, sizeof tmp, fmt, ap);
        va_end(ap);
        s += tmp;
    }
};

std::string lit(double x) {
    char b[64];
    snprintf(b, sizeof b, "%a", x);
    return b;
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
__device__ __forceinline__ d2 ldcs(const d2 *p) {
    d2 r;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcs(d2 *p, d2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int swz(int l) { return l ^ ((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7; }
)";

int swz_h(int l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7); }

unsigned xcombo_h(const uint16_t *s, int i) {
    unsigned r = 0;
    for (int k = 0; k < FSLOTS; ++k)
        if ((i >> k) & 1) r ^= s[k];
    return r;
}
int64_t xcombo_g(const int64_t *s, int i) {
    int64_t r = 0;
    for (int k = 0; k < FSLOTS; ++k)
        if ((i >> k) & 1) r ^= s[k];
    return r;
}
unsigned slot_pat(int s) {
    unsigned m = 0;
    for (int i = 0; i < FREGS; ++i)
        if ((i >> s) & 1) m |= 1u << i;
    return m;
}

// one gate as straight-line code over v[0..15]
void emit_gate(Out &o, const FGate &g) {
    const double2 *m = g.m;
    const int op = g.op;
    const bool thread_ctl = g.cl >= 0;
    if (thread_ctl) o("if ((tid >> %d) & 1) {\n", g.cl);
    if (op < FOP_DIAG) {
        const int kind = (op >> 1) / FSLOTS, s = (op >> 1) % FSLOTS, ctrl = op & 1;
        for (int i = 0; i < FREGS; ++i) {
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
        const int ctrl = code & 1, tpos = (code >> 1) % (FSLOTS + 1), var = (code >> 1) / (FSLOTS + 1);
        auto mul = [&](int i, const double2 &d) {
            if (var == FD_Z && d.x == -1.0)
                o("v[%d] = mk(-v[%d].x, -v[%d].y);\n", i, i, i);
            else
                o("v[%d] = cm(%s, %s, v[%d]);\n", i, lit(d.x).c_str(), lit(d.y).c_str(), i);
        };
        const bool d0_one = var != FD_GENERAL;
        if (tpos == FSLOTS) {  // target on a thread bit: one factor per thread
            o("if ((tid >> %d) & 1) {\n", g.tl);
            for (int i = 0; i < FREGS; ++i)
                if (!ctrl || ((g.cmask >> i) & 1)) mul(i, m[3]);
            o("}");
            if (!d0_one) {
                o(" else {\n");
                for (int i = 0; i < FREGS; ++i)
                    if (!ctrl || ((g.cmask >> i) & 1)) mul(i, m[0]);
                o("}");
            }
            o("\n");
        } else {
            for (int i = 0; i < FREGS; ++i) {
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

}  // namespace

std::string jit_source(const FPass &P, bool fma) {
    Out o;
    o("#define SVB_FMA %d\n", fma ? 1 : 0);
    o.s += kPreamble;
    const int nrows = FTILE >> P.flow;
    const int colmask = (1 << P.flow) - 1;
    o("extern \"C\" __global__ void __launch_bounds__(%d, %d) kpass(d2 *__restrict__ a, i64 ntiles) {\n",
      FTHREADS, FCTAS_PER_SM);
    o("__shared__ alignas(16) d2 buf[%d];\n__shared__ i64 rowoff[%d];\n", FTILE, nrows);
    o("const int tid = threadIdx.x;\nunsigned char *sb = reinterpret_cast<unsigned char *>(buf);\n");
    o("for (int r = tid; r < %d; r += %d) { i64 off = 0;\n", nrows, FTHREADS);
    for (int j = 0; j < FM - P.flow; ++j) o("if ((r >> %d) & 1) off |= 1ll << %d;\n", j, P.rowbit[j]);
    o("rowoff[r] = off; }\n__syncthreads();\n");
    o("for (i64 tix = blockIdx.x; tix < ntiles; tix += gridDim.x) {\ni64 base = 0;\n");
    for (int j = 0; j < P.ncomp; ++j) o("base |= ((tix >> %d) & 1) << %d;\n", j, P.comp[j]);
    if (!P.direct_first) {
        o("#pragma unroll\nfor (int k = 0; k < %d; ++k) { int e = tid + k * %d;\n", FREGS, FTHREADS);
        o("cpa(&buf[swz(e)], &a[base + rowoff[e >> %d] + (e & %d)]); }\n", P.flow, colmask);
        o("asm volatile(\"cp.async.commit_group;\\ncp.async.wait_group 0;\\n\" ::: \"memory\");\n__syncthreads();\n");
    }
    o("d2 v[%d];\n", FREGS);
    for (int gi = 0; gi < P.ngroups; ++gi) {
        const FGroup &G = P.groups[gi];
        const bool last = gi == P.ngroups - 1;
        o("{ // group %d\n", gi);
        if (gi == 0 && P.direct_first) {
            o("i64 g0 = %lldll;\n", (long long)P.gl_b);
            for (int j = 0; j < FTBITS; ++j) o("if ((tid >> %d) & 1) g0 ^= %lldll;\n", j, (long long)P.gl_t[j]);
            for (int i = 0; i < FREGS; ++i)
                o("v[%d] = ldcs(a + (base | (g0 ^ %lldll)));\n", i, (long long)xcombo_g(P.gl_s, i));
        } else {
            o("unsigned a0 = %uu;\n", (unsigned)G.ld_b);
            for (int j = 0; j < FTBITS; ++j) o("if ((tid >> %d) & 1) a0 ^= %uu;\n", j, (unsigned)G.ld_t[j]);
            for (int i = 0; i < FREGS; ++i)
                o("v[%d] = *reinterpret_cast<const d2 *>(sb + (a0 ^ %uu));\n", i, xcombo_h(G.ld_s, i));
        }
        for (int q = G.first; q < G.first + G.count; ++q) emit_gate(o, P.gates[q]);
        if (last && P.direct_last) {
            if (G.perm && gi == 0 && P.direct_first) o("__syncthreads();\n");
            o("i64 s0 = %lldll;\n", (long long)P.gs_b);
            for (int j = 0; j < FTBITS; ++j) o("if ((tid >> %d) & 1) s0 ^= %lldll;\n", j, (long long)P.gs_t[j]);
            for (int i = 0; i < FREGS; ++i)
                o("stcs(a + (base | (s0 ^ %lldll)), v[%d]);\n", (long long)xcombo_g(P.gs_s, i), i);
        } else {
            if (G.perm) o("__syncthreads();\n");
            o("unsigned b0 = %uu;\n", (unsigned)G.st_b);
            for (int j = 0; j < FTBITS; ++j) o("if ((tid >> %d) & 1) b0 ^= %uu;\n", j, (unsigned)G.st_t[j]);
            for (int i = 0; i < FREGS; ++i)
                o("*reinterpret_cast<d2 *>(sb + (b0 ^ %uu)) = v[%d];\n", xcombo_h(G.st_s, i), i);
            o("__syncthreads();\n");
        }
        o("}\n");
    }
    if (!P.direct_last) {
        o("#pragma unroll\nfor (int k = 0; k < %d; ++k) { int e = tid + k * %d;\n", FREGS, FTHREADS);
        o("a[base + rowoff[e >> %d] + (e & %d)] = buf[swz(e)]; }\n", P.flow, colmask);
    }
    o("__syncthreads();\n}\n}\n");
    return o.s;
}

// ---------------------------------------------------------------------------
// compile + cache

struct JitFn {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
};

static std::mutex g_jit_mu;
static std::unordered_map<uint64_t, JitFn> g_jit_cache;
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
    create_t create = nullptr;
    compile_t compile = nullptr;
    size_t_ log_size = nullptr, cubin_size = nullptr;
    get_t log = nullptr, cubin = nullptr;
    destroy_t destroy = nullptr;
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
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        return r;
    }();
    return n;
}

static bool nvrtc_compile(const std::string &src, std::vector<char> &cubin, std::string &log) {
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
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-fmad=false"};
    if (nv.compile(prog, 4, opts) != 0) {
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

// Compile (or fetch) one kernel per pass.  Returns false and leaves
// `fns` empty on any failure (the caller falls back to k_fused).
bool jit_build(const std::vector<FPass> &passes, bool fma, std::vector<void *> &fns) {
    fns.assign(passes.size(), nullptr);
    std::vector<std::string> srcs(passes.size());
    std::vector<uint64_t> keys(passes.size());
    std::vector<size_t> todo;
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        for (size_t i = 0; i < passes.size(); ++i) {
            srcs[i] = jit_source(passes[i], fma);
            keys[i] = hash_str(srcs[i]);
            auto it = g_jit_cache.find(keys[i]);
            if (it != g_jit_cache.end())
                fns[i] = it->second.fn;
            else
                todo.push_back(i);
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
            return false;
        }
        std::lock_guard<std::mutex> lk(g_jit_mu);
        for (size_t i : todo) {
            JitFn f;
            if (cudaLibraryLoadData(&f.lib, cubins[i].data(), nullptr, nullptr, 0, nullptr, nullptr, 0) !=
                    cudaSuccess ||
                cudaLibraryGetKernel(&f.fn, f.lib, "kpass") != cudaSuccess) {
                cudaGetLastError();
                fns.clear();
                return false;
            }
            g_jit_cache[keys[i]] = f;
            fns[i] = (void *)f.fn;
        }
    }
    return true;
}

// Host-only check: generate and NVRTC-compile every pass (no device needed).
int jit_compile_only(const std::vector<FPass> &passes, bool fma, std::string &err) {
    const char *dump = getenv("SVB_JIT_DUMP");  // directory: write pass sources and cubins
    int k = 0;
    for (const FPass &P : passes) {
        std::vector<char> cubin;
        std::string src = jit_source(P, fma);
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

bool jit_launch(void *fn, double2 *a, int64_t ntiles, int grid, cudaStream_t s) {
    long long nt = ntiles;
    void *args[] = {&a, &nt};
    return cudaLaunchKernel((const void *)fn, dim3(grid), dim3(FTHREADS), args, 0, s) == cudaSuccess;
}

}  // namespace svb
