"""Host emulator for the runtime-specialised pass kernels (debugging aid).

Compiles every pass source that SVB_JIT_DUMP wrote (passN.cu) as plain C++
with g++ -- one std::thread per CUDA thread of a single CTA, __syncthreads
as a std::barrier, cp.async as a synchronous copy -- and runs the passes in
order over a numpy state, so generated code can be checked against the
oracle without a GPU.

    python tools/jit_emu.py DUMP_DIR N_QUBITS [--ops-prefix K]

Used as a library by tests/test_jit_emu.py.
"""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np

SHIM = r"""
#include <atomic>
#include <barrier>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
typedef long long i64;
struct alignas(16) d2 { double x, y; };
static inline d2 mk(double x, double y) { d2 r; r.x = x; r.y = y; return r; }
static inline double __fma_rn(double a, double b, double c) { return std::fma(a, b, c); }
static inline double __dmul_rn(double a, double b) { return a * b; }
static inline double __dadd_rn(double a, double b) { return a + b; }
static inline double __dsub_rn(double a, double b) { return a - b; }
#if SVB_FMA
static inline d2 cm(double ar, double ai, d2 b) {
    return mk(__fma_rn(ar, b.x, -__dmul_rn(ai, b.y)), __fma_rn(ar, b.y, __dmul_rn(ai, b.x)));
}
static inline d2 row(double ar, double ai, d2 lo, double br, double bi, d2 hi) {
    return mk(__fma_rn(ar, lo.x, __fma_rn(-ai, lo.y, __fma_rn(br, hi.x, -__dmul_rn(bi, hi.y)))),
              __fma_rn(ar, lo.y, __fma_rn(ai, lo.x, __fma_rn(br, hi.y, __dmul_rn(bi, hi.x)))));
}
static inline d2 rrow(double a, d2 lo, double b, d2 hi) {
    return mk(__fma_rn(a, lo.x, __dmul_rn(b, hi.x)), __fma_rn(a, lo.y, __dmul_rn(b, hi.y)));
}
static inline d2 rirow(double a, d2 r, double s, d2 im) {
    return mk(__fma_rn(a, r.x, -__dmul_rn(s, im.y)), __fma_rn(a, r.y, __dmul_rn(s, im.x)));
}
#else
static inline d2 cm(double ar, double ai, d2 b) {
    return mk(__dsub_rn(__dmul_rn(ar, b.x), __dmul_rn(ai, b.y)), __dadd_rn(__dmul_rn(ar, b.y), __dmul_rn(ai, b.x)));
}
static inline d2 row(double ar, double ai, d2 lo, double br, double bi, d2 hi) {
    d2 p = cm(ar, ai, lo), q = cm(br, bi, hi);
    return mk(__dadd_rn(p.x, q.x), __dadd_rn(p.y, q.y));
}
static inline d2 rrow(double a, d2 lo, double b, d2 hi) {
    return mk(__dadd_rn(__dmul_rn(a, lo.x), __dmul_rn(b, hi.x)), __dadd_rn(__dmul_rn(a, lo.y), __dmul_rn(b, hi.y)));
}
static inline d2 rirow(double a, d2 r, double s, d2 im) {
    return mk(__dadd_rn(__dmul_rn(a, r.x), -__dmul_rn(s, im.y)), __dadd_rn(__dmul_rn(a, r.y), __dmul_rn(s, im.x)));
}
#endif
static inline void cpa(void *smem, const void *g) { std::memcpy(smem, g, 16); }
static inline d2 ldcs(const d2 *p) { return *p; }
static inline void stcs(d2 *p, d2 v) { *p = v; }
static inline int swz(int l) { return l ^ ((l >> 3) ^ (l >> 6) ^ (l >> 9) ^ (l >> 12)) & 7; }
static inline double ng(double x) { return -x; }
static inline int __double2hiint(double x) { uint64_t b; std::memcpy(&b, &x, 8); return (int)(b >> 32); }
static inline double cneg(double x, unsigned m) {
    uint64_t b; std::memcpy(&b, &x, 8); b ^= uint64_t(m) << 32; std::memcpy(&x, &b, 8); return x;
}
// tile ring (mode 3): cp.async is a synchronous copy here, so an mbarrier
// only counts arrivals and flips its phase; warpgroup barriers are barriers
// over the warpgroup's threads
struct EmuMbar { std::atomic<unsigned> count{0}, phase{0}; unsigned expected = 0; };
static EmuMbar g_mbar[3];
static void mb_init(EmuMbar *m, unsigned c) { m->expected = c; m->count = 0; m->phase = 0; }
static void mb_arrive_cp(EmuMbar *m) {
    if (m->count.fetch_add(1) + 1 == m->expected) { m->count = 0; m->phase.fetch_add(1); }
}
static void mb_wait(EmuMbar *m, unsigned parity) { while ((m->phase.load() & 1) == parity) std::this_thread::yield(); }
static std::barrier<> *g_wgbar[2];
static void wg_sync(int wg, int) { g_wgbar[wg]->arrive_and_wait(); }
static thread_local int t_tid;
static int g_bid, g_grid;
static d2 *g_smem;
static std::barrier<> *g_bar;
"""

DRIVER = r"""
// CTAs one after another (blocks of one pass touch disjoint tiles)
extern "C" void emu_run(d2 *a, long long ntiles, int nthreads, int grid) {
    std::vector<d2> sm(2 << 13);
    g_smem = sm.data();
    std::barrier<> bar(nthreads);
    g_bar = &bar;
    std::barrier<> wb0(nthreads / 2 > 0 ? nthreads / 2 : 1), wb1(nthreads / 2 > 0 ? nthreads / 2 : 1);
    g_wgbar[0] = &wb0;
    g_wgbar[1] = &wb1;
    g_grid = grid;
    for (g_bid = 0; g_bid < grid; ++g_bid) {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t) th.emplace_back([=] { t_tid = t; kpass_body(a, ntiles); });
        for (auto &x : th) x.join();
    }
}
"""


def translate(src: str):
    """CUDA pass source -> (C++ source, threads per CTA)."""
    fma = "#define SVB_FMA 1" in src
    body = src[src.index("__constant__ double kc"):]
    m = re.search(r'extern "C" __global__ void __launch_bounds__\((\d+), (\d+)\) kpass\(', body)
    nthreads = int(m.group(1))
    body = body.replace(m.group(0), "static void kpass_body(")
    body = body.replace("__constant__ ", "")
    body = re.sub(r"extern __shared__ d2 dsm\[\];", "d2 *dsm = g_smem;", body)
    body = re.sub(r"__shared__ alignas\(16\) d2 dsm\[\d+\];", "d2 *dsm = g_smem;", body)
    body = body.replace("threadIdx.x", "t_tid").replace("blockIdx.x", "g_bid").replace("gridDim.x", "g_grid")
    body = body.replace("__syncthreads()", "g_bar->arrive_and_wait()")
    body = body.replace("__popc(", "__builtin_popcount(")
    body = re.sub(r'asm volatile\("" : "\+r"\(tg\)\);', "", body)
    body = re.sub(r'asm volatile\("cp\.async\.[a-z_]+(?: 0)?;\\n" ::: "memory"\);', "", body)
    # a group's shared-memory stores may overwrite chunks that other lanes of
    # the same warp have not loaded yet (the row swizzle changes between
    # transitions): the device kernel orders them with __syncwarp(); the
    # emulator's threads are independent, so order them with the barrier
    ring = "__shared__ unsigned long long mbar[3];" in body
    # (ring: the two warpgroups run out of phase -- their own barrier)
    body = body.replace("__syncwarp();", "wg_sync(wg, 0);" if ring else "g_bar->arrive_and_wait();")
    body = body.replace("__shared__ unsigned long long mbar[3];", "EmuMbar *mbar = g_mbar;")
    nregs = int(re.search(r"d2 v\[(\d+)\];", body).group(1))
    tile = (nthreads // 2 if ring else nthreads) * nregs  # ring: two warpgroups, one tile each
    return f"#define SVB_FMA {1 if fma else 0}\n" + SHIM + body + DRIVER, tile


def build(path_cu: str, out_dir: str):
    cpp, tile = translate(open(path_cu).read())
    nthreads = int(re.search(r"__launch_bounds__\((\d+)", open(path_cu).read()).group(1))
    base = os.path.join(out_dir, os.path.basename(path_cu)[:-3])
    open(base + ".cpp", "w").write(cpp)
    subprocess.run(["g++", "-std=c++20", "-O1", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                    base + ".cpp", "-o", base + ".so"], check=True)
    lib = ctypes.CDLL(base + ".so")
    lib.emu_run.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int]
    return lib, nthreads, tile


def run_passes(dump_dir: str, state: np.ndarray, out_dir=None, grid=1):
    """Run pass0.cu, pass1.cu, ... of dump_dir in order over `state` (in place)
    with `grid` CTAs (each loops over tiles blockIdx, blockIdx + grid, ...);
    returns the state after each pass."""
    out_dir = out_dir or dump_dir
    a = state
    assert a.flags.c_contiguous and a.dtype == np.complex128
    snaps = []
    i = 0
    while os.path.exists(os.path.join(dump_dir, f"pass{i}.cu")):
        lib, nthreads, tile = build(os.path.join(dump_dir, f"pass{i}.cu"), out_dir)
        ntiles = len(a) // tile
        lib.emu_run(a.ctypes.data, ntiles, nthreads, min(grid, ntiles))
        snaps.append(a.copy())
        i += 1
    return snaps


if __name__ == "__main__":
    print(translate(open(sys.argv[1]).read())[0][:200])
