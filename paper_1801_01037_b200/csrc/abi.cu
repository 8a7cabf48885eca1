// abi.cu -- the extern "C" boundary (include/svb.h) and the partitioned-state
// runtime (svb_dist).
//
// Validation mirrors the reference wrapper (kernel/__init__.py:83-97,
// 124-128): power-of-two length >= 2, 2^(t+1) <= size, control in range and
// != target.  Failures return SVB_EINVAL with a message; nothing is launched.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/svb.h"
#include "svb_common.cuh"

namespace svb {

LaunchInfo launch_gate(double2 *a, int64_t n_amps, const Gate &g, int t, int c, cudaStream_t s);
LaunchInfo launch_dense_embed(double2 *u, int64_t dim, const Gate &g, int t, int c, cudaStream_t s);
LaunchInfo launch_signal(unsigned *flag, unsigned value, cudaStream_t s);
LaunchInfo launch_peer_copy(double2 *dst, const double2 *src, int64_t count, cudaStream_t s);
LaunchInfo launch_peer_swap_half(double2 *a, double2 *b, int64_t begin, int64_t end, int bit, int va, int vb,
                                 cudaStream_t s);
LaunchInfo launch_dense_matvec(const double2 *u, const double2 *x, double2 *y, int64_t dim, int64_t row0,
                               int64_t nrows, cudaStream_t s);
int launch_norm2(const double2 *a, int64_t n, double *scratch, cudaStream_t s);
int norm_scratch_doubles();
int launch_probs(const double2 *a, int64_t n, double *p, cudaStream_t s);
int launch_permute(const double2 *src, double2 *dst, int64_t n, const int *p2l, int nbits, cudaStream_t s);
LaunchInfo launch_exchange_own_row(double2 *own, const double2 *other, int64_t count, const Gate &g,
                                   int own_is_low, int cbit, int64_t offset, cudaStream_t s);
LaunchInfo launch_pair_update(double2 *lo_slab, double2 *hi_slab, int64_t begin, int64_t end,
                              const Gate &g, int cbit, cudaStream_t s);
LaunchInfo launch_pack_half(const double2 *src, double2 *dst, int64_t count, int bit, int value, int64_t offset,
                            cudaStream_t s);
LaunchInfo launch_unpack_half(double2 *dst, const double2 *src, int64_t count, int bit, int value, int64_t offset,
                              cudaStream_t s);
LaunchInfo launch_pack_ctrl(const double2 *src, double2 *dst, int64_t count, int cbit, int64_t offset,
                            cudaStream_t s);
LaunchInfo launch_exchange_packed(double2 *own, const double2 *other, int64_t count, const Gate &g,
                                  int own_is_low, int cbit, int64_t offset, cudaStream_t s);
int run_ops_device(double2 *a, int64_t n_amps, const svb_op *ops, int nops, unsigned flags,
                   cudaStream_t s, int64_t *launches);
int plan_passes(int n, const svb_op *ops, int nops, unsigned flags, int *groups);
int jit_check(int n, const svb_op *ops, int nops, unsigned flags);
struct SwapNet;
int swap_suffix(int n, const svb_op *ops, int nops, SwapNet *out);

static thread_local char g_err[512];
std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char *where) {
    set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SVB_ENOMEM : SVB_ECUDA;
}

// ---- launch profiler -------------------------------------------------------
struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    int64_t bytes;
};
static std::mutex g_prof_mu;
static bool g_prof_enabled = false;
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_prof_pool;
static cudaEvent_t g_prof_pending = nullptr;
static double g_prof_ms[PROF_NCLASSES];
static int64_t g_prof_n[PROF_NCLASSES], g_prof_bytes[PROF_NCLASSES];

static cudaEvent_t prof_event() {
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

bool prof_on() { return g_prof_enabled; }

void prof_begin(cudaStream_t s) {
    if (!g_prof_enabled) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_pending = prof_event();
    cudaEventRecord(g_prof_pending, s);
}

void prof_end(cudaStream_t s, const LaunchInfo &li) {
    if (!g_prof_enabled || !g_prof_pending) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, s);
    g_prof_recs.push_back(ProfRec{g_prof_pending, b, li.cls, li.alg_bytes});
    g_prof_pending = nullptr;
}

// fold finished records into the per-class totals (synchronises on events)
static void prof_drain() {
    for (auto &r : g_prof_recs) {
        float ms = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&ms, r.a, r.b);
        g_prof_ms[r.cls] += ms;
        g_prof_n[r.cls] += 1;
        g_prof_bytes[r.cls] += r.bytes;
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    g_prof_recs.clear();
}

static int log2_exact(int64_t n) {
    if (n < 2 || (n & (n - 1))) return -1;
    int b = 0;
    while ((int64_t(1) << b) < n) ++b;
    return b;
}

static int check_amps(const void *amps, int64_t n_amps) {
    if (!amps) {
        set_error("amplitude pointer is NULL");
        return SVB_EINVAL;
    }
    if (log2_exact(n_amps) < 0) {
        set_error("amplitude count must be a power of two >= 2, got %lld", (long long)n_amps);
        return SVB_EINVAL;
    }
    if (reinterpret_cast<uintptr_t>(amps) % 16) {
        set_error("amplitude buffer must be 16-byte aligned");
        return SVB_EINVAL;
    }
    return SVB_OK;
}

static int check_target(int t, int64_t n_amps) {  // kernel/__init__.py:95-97
    if (t < 0 || t > 62 || (int64_t(2) << t) > n_amps) {
        set_error("qubit %d out of range for %lld amplitudes", t, (long long)n_amps);
        return SVB_EINVAL;
    }
    return SVB_OK;
}

static int check_control(int c, int t, int64_t n_amps) {  // kernel/__init__.py:124-128
    if (c < 0 || c > 62 || (int64_t(1) << c) >= n_amps) {
        set_error("control %d out of range for %lld amplitudes", c, (long long)n_amps);
        return SVB_EINVAL;
    }
    if (c == t) {
        set_error("control and target must differ");
        return SVB_EINVAL;
    }
    return SVB_OK;
}

int check_ops(int n, const svb_op *ops, int nops) {
    if (nops < 0 || (nops > 0 && !ops)) {
        set_error("bad op list");
        return SVB_EINVAL;
    }
    int64_t n_amps = int64_t(1) << n;
    for (int i = 0; i < nops; ++i) {
        const svb_op &o = ops[i];
        if (o.kind != 0 && o.kind != 1) {
            set_error("op %d: unknown kind %d", i, o.kind);
            return SVB_EINVAL;
        }
        int r = check_target(o.target, n_amps);
        if (r == SVB_OK && o.kind == 1) r = check_control(o.control, o.target, n_amps);
        if (r != SVB_OK) return r;
    }
    return SVB_OK;
}

// Grow-only device staging buffer for the host-buffer entry points.
struct Staging {
    std::mutex mu;
    void *ptr = nullptr;
    size_t bytes = 0;
    int device = -1;
};
static Staging g_stage;

// The single-gate host seam (svsim's backend contract: one gate per call on
// a caller-owned host array) streamed through the device in units instead
// of one whole-state H2D, kernel, D2H: a unit is one block of 2^s
// amplitudes (target t < s) or the two blocks b, b ^ 2^(t-s) a pair spans
// (t >= s; in the staging slot the partner sits at distance 2^s, so the
// kernel runs with target s).  Three slots on three streams: the H2D of one
// unit overlaps the kernel and the D2H of the others (PCIe both ways at
// once when the host array is pinned or registered, svb_host_register).  A
// control bit c >= s is constant over a unit: units whose control bit is 0
// are not copied at all.  Same kernels, same arithmetic: bit-identical.
struct SeamPipe {
    int device = -1;
    double2 *buf = nullptr;  // 3 slots x 2^(s+1) amplitudes
    int64_t slot_amps = 0;
    cudaStream_t st[3] = {nullptr, nullptr, nullptr};
};
static SeamPipe g_seam;
constexpr int kSeamBits = 22;  // 64 MiB blocks

static int seam_apply(double *host, int64_t n_amps, const double q[8], int c, int t) {
    int n = 0;
    while ((int64_t(1) << n) < n_amps) ++n;
    const int s = std::min(kSeamBits, n - 3);
    int d;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    const int64_t S = int64_t(1) << s;
    if (g_seam.buf && (g_seam.device != d || g_seam.slot_amps < 2 * S)) {
        int cur = d;
        cudaSetDevice(g_seam.device);
        cudaFree(g_seam.buf);
        for (auto &x : g_seam.st) cudaStreamDestroy(x);
        cudaSetDevice(cur);
        g_seam = SeamPipe();
    }
    if (!g_seam.buf) {
        e = cudaMalloc((void **)&g_seam.buf, size_t(3) * 2 * S * sizeof(double2));
        if (e != cudaSuccess) {
            g_seam.buf = nullptr;
            return cuda_status(e, "seam staging cudaMalloc");
        }
        for (auto &x : g_seam.st) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
        g_seam.slot_amps = 2 * S;
        g_seam.device = d;
    }
    double2 *h = reinterpret_cast<double2 *>(host);
    const Gate g = make_gate(q);
    const bool pair = t >= s;
    const int64_t nblocks = n_amps >> s;
    int64_t u = 0;
    for (int64_t b = 0; b < nblocks; ++b) {
        if (pair && ((b >> (t - s)) & 1)) continue;  // the upper block of a pair
        if (c >= s && !((b >> (c - s)) & 1)) continue;  // control clear over the whole unit
        const int k = int(u++ % 3);
        cudaStream_t st = g_seam.st[k];
        double2 *slot = g_seam.buf + k * 2 * S;
        const int64_t b2 = pair ? (b | (int64_t(1) << (t - s))) : -1;
        e = cudaMemcpyAsync(slot, h + b * S, S * sizeof(double2), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && pair)
            e = cudaMemcpyAsync(slot + S, h + b2 * S, S * sizeof(double2), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_status(e, "seam H2D");
        prof_begin(st);
        LaunchInfo li = launch_gate(slot, pair ? 2 * S : S, g, pair ? s : t, c >= 0 && c < s ? c : -1, st);
        prof_end(st, li);
        g_launches += li.kernels;
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e, "seam kernel");
        e = cudaMemcpyAsync(h + b * S, slot, S * sizeof(double2), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && pair)
            e = cudaMemcpyAsync(h + b2 * S, slot + S, S * sizeof(double2), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return cuda_status(e, "seam D2H");
    }
    for (auto &x : g_seam.st) {
        e = cudaStreamSynchronize(x);
        if (e != cudaSuccess) return cuda_status(e, "seam sync");
    }
    return SVB_OK;
}

// below this size the whole state goes in one copy each way
constexpr int64_t kSeamMinAmps = int64_t(1) << 22;

}  // namespace svb

using namespace svb;

extern "C" {

int svb_abi_version(void) { return 1; }

const char *svb_last_error(void) { return g_err; }

int64_t svb_launch_count(void) { return g_launches.load(); }

int svb_apply_1q(void *amps, int64_t n_amps, const double q[8], int target, void *stream) {
    int r = check_amps(amps, n_amps);
    if (r == SVB_OK) r = check_target(target, n_amps);
    if (r != SVB_OK) return r;
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_gate((double2 *)amps, n_amps, make_gate(q), target, -1, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_apply_1q");
    return SVB_OK;
}

int svb_apply_c1q(void *amps, int64_t n_amps, const double q[8], int control, int target,
                  void *stream) {
    int r = check_amps(amps, n_amps);
    if (r == SVB_OK) r = check_target(target, n_amps);
    if (r == SVB_OK) r = check_control(control, target, n_amps);
    if (r != SVB_OK) return r;
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_gate((double2 *)amps, n_amps, make_gate(q), target, control,
                                (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_apply_c1q");
    return SVB_OK;
}

int svb_run_ops(void *amps, int64_t n_amps, const svb_op *ops, int nops, unsigned flags,
                void *stream) {
    int r = check_amps(amps, n_amps);
    if (r != SVB_OK) return r;
    int n = log2_exact(n_amps);
    if ((r = check_ops(n, ops, nops)) != SVB_OK) return r;
    int64_t launches = 0;
    r = run_ops_device((double2 *)amps, n_amps, ops, nops, flags, (cudaStream_t)stream, &launches);
    g_launches += launches;
    if (r != SVB_OK) return r;
    SVB_CHECK_LAUNCH("svb_run_ops");
    return SVB_OK;
}

int svb_jit_check(int n_qubits, const svb_op *ops, int nops, unsigned flags, int *compiled) {
    if (n_qubits < 1 || n_qubits > 62 || !compiled) {
        set_error("bad arguments to svb_jit_check");
        return SVB_EINVAL;
    }
    int r = check_ops(n_qubits, ops, nops);
    if (r != SVB_OK) return r;
    int c = jit_check(n_qubits, ops, nops, flags);
    if (c < 0) return SVB_ESTATE;
    *compiled = c;
    return SVB_OK;
}

int svb_swap_suffix(int n_qubits, const svb_op *ops, int nops) {
    if (n_qubits < 1 || n_qubits > 62 || check_ops(n_qubits, ops, nops) != SVB_OK) return 0;
    return swap_suffix(n_qubits, ops, nops, nullptr);
}

int svb_plan_passes(int n_qubits, const svb_op *ops, int nops, unsigned flags, int *passes,
                    int *groups) {
    if (n_qubits < 1 || n_qubits > 62 || !passes) {
        set_error("bad arguments to svb_plan_passes");
        return SVB_EINVAL;
    }
    int r = check_ops(n_qubits, ops, nops);
    if (r != SVB_OK) return r;
    *passes = plan_passes(n_qubits, ops, nops, flags, groups);
    return SVB_OK;
}

int svb_norm2(const void *amps, int64_t n_amps, double *out, void *stream) {
    int r = check_amps(amps, n_amps);
    if (r != SVB_OK) return r;
    if (!out) {
        set_error("out is NULL");
        return SVB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    double *scratch = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&scratch, sizeof(double) * norm_scratch_doubles(), s);
    if (e != cudaSuccess) return cuda_status(e, "svb_norm2 alloc");
    g_launches += launch_norm2((const double2 *)amps, n_amps, scratch, s);  // not profiled
    e = cudaMemcpyAsync(out, scratch + norm_scratch_doubles() - 1, sizeof(double),
                        cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(scratch, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "svb_norm2");
    return SVB_OK;
}

int svb_dense_embed(void *u, int n_qubits, const double q[8], int control, int target, void *stream) {
    if (!u || !q || n_qubits < 1 || n_qubits > SVB_MAX_DENSE_QUBITS) {
        set_error("dense embed: n_qubits %d outside [1, %d] or NULL buffer", n_qubits, SVB_MAX_DENSE_QUBITS);
        return n_qubits > SVB_MAX_DENSE_QUBITS ? SVB_ENOMEM : SVB_EINVAL;
    }
    if (target < 0 || target >= n_qubits || control >= n_qubits || control == target || control < -1) {
        set_error("dense embed: control %d / target %d invalid for n=%d", control, target, n_qubits);
        return SVB_EINVAL;
    }
    const int64_t dim = int64_t(1) << n_qubits;
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_dense_embed((double2 *)u, dim, make_gate(q), target, control, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_dense_embed");
    return SVB_OK;
}

int svb_dense_matvec(const void *u, const void *x, void *y, int64_t dim, int64_t row0, int64_t nrows,
                     void *stream) {
    if (!u || !x || !y || dim < 1 || (dim & (dim - 1)) || dim > (int64_t(1) << SVB_MAX_DENSE_QUBITS) ||
        row0 < 0 || nrows < 0 || row0 + nrows > dim) {
        set_error("dense matvec: dim %lld, rows [%lld, %lld) invalid", (long long)dim, (long long)row0,
                  (long long)(row0 + nrows));
        return SVB_EINVAL;
    }
    if (nrows == 0) return SVB_OK;
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_dense_matvec((const double2 *)u, (const double2 *)x, (double2 *)y, dim, row0, nrows,
                                        (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_dense_matvec");
    return SVB_OK;
}

int svb_probs(const void *amps, int64_t n_amps, double *probs, void *stream) {
    int r = check_amps(amps, n_amps);
    if (r != SVB_OK) return r;
    if (!probs) {
        set_error("probs is NULL");
        return SVB_EINVAL;
    }
    g_launches += launch_probs((const double2 *)amps, n_amps, probs, (cudaStream_t)stream);
    SVB_CHECK_LAUNCH("svb_probs");
    return SVB_OK;
}

int svb_exchange_own_row(void *own, const void *other, int64_t count, const double q[8],
                         int own_is_low, int cbit, int64_t index_offset, void *stream) {
    if (!own || !other || count < 0 || cbit > 62 || index_offset < 0) {
        set_error("bad arguments to svb_exchange_own_row");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_exchange_own_row((double2 *)own, (const double2 *)other, count,
                                            make_gate(q), own_is_low, cbit, index_offset,
                                            (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_exchange_own_row");
    return SVB_OK;
}

int svb_permute_qubits(const void *src, void *dst, int64_t n_amps, const int *phys_to_logical, int n,
                       void *stream) {
    int r = check_amps(src, n_amps);
    if (r == SVB_OK) r = check_amps(dst, n_amps);
    if (r != SVB_OK) return r;
    if (!phys_to_logical || n != log2_exact(n_amps) || src == dst) {
        set_error("bad arguments to svb_permute_qubits (needs n = log2(n_amps), out of place)");
        return SVB_EINVAL;
    }
    uint64_t seen = 0;
    for (int j = 0; j < n; ++j) {
        int q = phys_to_logical[j];
        if (q < 0 || q >= n || ((seen >> q) & 1)) {
            set_error("phys_to_logical is not a permutation of 0..%d", n - 1);
            return SVB_EINVAL;
        }
        seen |= uint64_t(1) << q;
    }
    g_launches += launch_permute((const double2 *)src, (double2 *)dst, n_amps, phys_to_logical, n,
                                 (cudaStream_t)stream);
    SVB_CHECK_LAUNCH("svb_permute_qubits");
    return SVB_OK;
}

int svb_pack_ctrl(const void *src, void *dst, int64_t count, int cbit, int64_t offset, void *stream) {
    if (!src || !dst || count < 0 || cbit < 0 || cbit > 62 || offset < 0) {
        set_error("bad arguments to svb_pack_ctrl");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_pack_ctrl((const double2 *)src, (double2 *)dst, count, cbit, offset,
                                     (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_pack_ctrl");
    return SVB_OK;
}

int svb_pack_half(const void *src, void *dst, int64_t count, int bit, int value, int64_t offset, void *stream) {
    if (!src || !dst || count < 0 || bit < 0 || bit > 62 || (value != 0 && value != 1) || offset < 0) {
        set_error("bad arguments to svb_pack_half");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_pack_half((const double2 *)src, (double2 *)dst, count, bit, value, offset,
                                     (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_pack_half");
    return SVB_OK;
}

int svb_unpack_half(void *dst, const void *src, int64_t count, int bit, int value, int64_t offset, void *stream) {
    if (!src || !dst || count < 0 || bit < 0 || bit > 62 || (value != 0 && value != 1) || offset < 0) {
        set_error("bad arguments to svb_unpack_half");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_unpack_half((double2 *)dst, (const double2 *)src, count, bit, value, offset,
                                       (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_unpack_half");
    return SVB_OK;
}

int svb_exchange_own_row_packed(void *own, const void *other_packed, int64_t count, const double q[8],
                                int own_is_low, int cbit, int64_t offset, void *stream) {
    if (!own || !other_packed || count < 0 || cbit < 0 || cbit > 62 || offset < 0) {
        set_error("bad arguments to svb_exchange_own_row_packed");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_exchange_packed((double2 *)own, (const double2 *)other_packed, count,
                                           make_gate(q), own_is_low, cbit, offset, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_exchange_own_row_packed");
    return SVB_OK;
}

int svb_pair_update(void *lo_slab, void *hi_slab, int64_t begin, int64_t end, const double q[8],
                    int cbit, void *stream) {
    if (!lo_slab || !hi_slab || begin < 0 || end < begin || cbit > 62) {
        set_error("bad arguments to svb_pair_update");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_pair_update((double2 *)lo_slab, (double2 *)hi_slab, begin, end,
                                       make_gate(q), cbit, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_pair_update");
    return SVB_OK;
}

int svb_peer_swap_half(void *a, void *b, int64_t begin, int64_t end, int bit, int va, int vb, void *stream) {
    if (!a || !b || begin < 0 || end < begin || bit < 0 || bit > 62 || (va & ~1) || (vb & ~1)) {
        set_error("bad arguments to svb_peer_swap_half");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_peer_swap_half((double2 *)a, (double2 *)b, begin, end, bit, va, vb, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_peer_swap_half");
    return SVB_OK;
}

int svb_stream_signal(void *flag, uint32_t value, void *stream) {
    if (!flag || (uintptr_t(flag) & 3)) {
        set_error("svb_stream_signal: flag must be a 4-byte aligned device address");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_signal((unsigned *)flag, value, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_stream_signal");
    return SVB_OK;
}

int svb_stream_wait(void *flag, uint32_t value, void *stream) {
    if (!flag || (uintptr_t(flag) & 3)) {
        set_error("svb_stream_wait: flag must be a 4-byte aligned device address");
        return SVB_EINVAL;
    }
    // cuStreamWaitValue32(stream, addr, value, CU_STREAM_WAIT_VALUE_GEQ)
    typedef int (*wait_t)(void *, unsigned long long, unsigned, unsigned);
    static wait_t wait = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return (wait_t)fn;
    }();
    if (!wait) {
        set_error("svb_stream_wait: cuStreamWaitValue32 unavailable");
        return SVB_ECUDA;
    }
    const int r = wait(stream, (unsigned long long)(uintptr_t)flag, value, 0u /* GEQ */);
    if (r != 0) {
        set_error("svb_stream_wait: cuStreamWaitValue32 failed (CUresult %d)", r);
        return SVB_ECUDA;
    }
    return SVB_OK;
}

int svb_host_register(void *host, int64_t bytes) {
    if (!host || bytes <= 0) {
        set_error("bad arguments to svb_host_register");
        return SVB_EINVAL;
    }
    cudaError_t e = cudaHostRegister(host, size_t(bytes), cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        return SVB_OK;
    }
    if (e != cudaSuccess) return cuda_status(e, "cudaHostRegister");
    return SVB_OK;
}

int svb_host_unregister(void *host) {
    cudaError_t e = cudaHostUnregister(host);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_status(e, "cudaHostUnregister");
    }
    return SVB_OK;
}

int svb_copy_async(void *dst, const void *src, int64_t bytes, void *stream) {
    if (!dst || !src || bytes < 0) {
        set_error("bad arguments to svb_copy_async");
        return SVB_EINVAL;
    }
    cudaError_t e = cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDefault, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "svb_copy_async");
    return SVB_OK;
}

int svb_peer_copy(void *dst, const void *src, int64_t n_amps, void *stream) {
    if (!dst || !src || n_amps < 0) {
        set_error("bad arguments to svb_peer_copy");
        return SVB_EINVAL;
    }
    prof_begin((cudaStream_t)stream);
    LaunchInfo li = launch_peer_copy((double2 *)dst, (const double2 *)src, n_amps, (cudaStream_t)stream);
    prof_end((cudaStream_t)stream, li);
    g_launches += li.kernels;
    SVB_CHECK_LAUNCH("svb_peer_copy");
    return SVB_OK;
}

int svb_ipc_handle(const void *dev_ptr, unsigned char handle[64], int64_t *offset) {
    if (!dev_ptr || !handle || !offset) {
        set_error("svb_ipc_handle: NULL argument");
        return SVB_EINVAL;
    }
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr));
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
    memcpy(handle, &h, 64);
    // the handle names the whole allocation (a caching allocator's segment);
    // the opener gets its base, so ship the buffer's offset in it
    typedef int (*range_t)(unsigned long long *, size_t *, unsigned long long);
    static range_t range = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return (range_t)fn;
    }();
    unsigned long long base = 0;
    size_t size = 0;
    if (!range || range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0) {
        set_error("svb_ipc_handle: cuMemGetAddressRange unavailable or failed");
        return SVB_ECUDA;
    }
    *offset = int64_t((uintptr_t)dev_ptr - base);
    return SVB_OK;
}

int svb_ipc_open(const unsigned char handle[64], void **dev_ptr) {
    if (!handle || !dev_ptr) {
        set_error("svb_ipc_open: NULL argument");
        return SVB_EINVAL;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcOpenMemHandle");
    return SVB_OK;
}

int svb_ipc_close(void *dev_ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcCloseMemHandle");
    return SVB_OK;
}

// ---- host-buffer entry points ---------------------------------------------

static int host_stage(double *host, int64_t n_amps, void **dev) {
    int d;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    size_t bytes = size_t(n_amps) * 16;
    if (g_stage.ptr && (g_stage.device != d || g_stage.bytes < bytes)) {
        int cur = d;
        cudaSetDevice(g_stage.device);
        cudaFree(g_stage.ptr);
        cudaSetDevice(cur);
        g_stage.ptr = nullptr;
        g_stage.bytes = 0;
    }
    if (!g_stage.ptr) {
        e = cudaMalloc(&g_stage.ptr, bytes);
        if (e != cudaSuccess) {
            g_stage.ptr = nullptr;
            return cuda_status(e, "staging cudaMalloc");
        }
        g_stage.bytes = bytes;
        g_stage.device = d;
    }
    e = cudaMemcpy(g_stage.ptr, host, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_status(e, "H2D");
    *dev = g_stage.ptr;
    return SVB_OK;
}

static int host_unstage(double *host, int64_t n_amps, const void *dev) {
    cudaError_t e = cudaMemcpy(host, dev, size_t(n_amps) * 16, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_status(e, "D2H");
    return SVB_OK;
}

int svb_host_apply_1q(double *host_amps, int64_t n_amps, const double q[8], int target) {
    int r = check_amps(host_amps, n_amps);
    if (r == SVB_OK) r = check_target(target, n_amps);
    if (r != SVB_OK) return r;
    std::lock_guard<std::mutex> lk(g_stage.mu);
    if (n_amps >= kSeamMinAmps) return seam_apply(host_amps, n_amps, q, -1, target);
    void *dev;
    if ((r = host_stage(host_amps, n_amps, &dev)) != SVB_OK) return r;
    if ((r = svb_apply_1q(dev, n_amps, q, target, nullptr)) != SVB_OK) return r;
    return host_unstage(host_amps, n_amps, dev);
}

int svb_host_apply_c1q(double *host_amps, int64_t n_amps, const double q[8], int control,
                       int target) {
    int r = check_amps(host_amps, n_amps);
    if (r == SVB_OK) r = check_target(target, n_amps);
    if (r == SVB_OK) r = check_control(control, target, n_amps);
    if (r != SVB_OK) return r;
    std::lock_guard<std::mutex> lk(g_stage.mu);
    if (n_amps >= kSeamMinAmps) return seam_apply(host_amps, n_amps, q, control, target);
    void *dev;
    if ((r = host_stage(host_amps, n_amps, &dev)) != SVB_OK) return r;
    if ((r = svb_apply_c1q(dev, n_amps, q, control, target, nullptr)) != SVB_OK) return r;
    return host_unstage(host_amps, n_amps, dev);
}

int svb_host_run_ops(const double *host_in, double *host_out, int64_t n_amps, const svb_op *ops,
                     int nops, unsigned flags) {
    int r = check_amps(host_in, n_amps);
    if (r == SVB_OK) r = check_amps(host_out, n_amps);
    if (r != SVB_OK) return r;
    if ((r = check_ops(log2_exact(n_amps), ops, nops)) != SVB_OK) return r;
    std::lock_guard<std::mutex> lk(g_stage.mu);
    void *dev;
    if ((r = host_stage(const_cast<double *>(host_in), n_amps, &dev)) != SVB_OK) return r;
    if ((r = svb_run_ops(dev, n_amps, ops, nops, flags, nullptr)) != SVB_OK) return r;
    return host_unstage(host_out, n_amps, dev);
}

// three device state buffers + three streams for svb_host_run_ops_batch
struct BatchStage {
    std::mutex mu;
    void *buf[3] = {nullptr, nullptr, nullptr};
    size_t bytes = 0;
    int device = -1;
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};  // H2D, compute, D2H
    cudaEvent_t in[3], ran[3], out[3];
};
static BatchStage g_batch;

static int batch_setup(size_t bytes) {
    int d;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    BatchStage &B = g_batch;
    if (B.device >= 0 && (B.device != d || B.bytes < bytes)) {
        int cur = d;
        cudaSetDevice(B.device);
        for (int i = 0; i < 3; ++i) {
            cudaFree(B.buf[i]);
            B.buf[i] = nullptr;
        }
        if (B.device != d) {
            for (int i = 0; i < 3; ++i) {
                cudaStreamDestroy(B.s[i]);
                cudaEventDestroy(B.in[i]);
                cudaEventDestroy(B.ran[i]);
                cudaEventDestroy(B.out[i]);
                B.s[i] = nullptr;
            }
        }
        cudaSetDevice(cur);
        B.bytes = 0;
    }
    if (!B.s[0]) {
        for (int i = 0; i < 3; ++i) {
            if ((e = cudaStreamCreateWithFlags(&B.s[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_status(e, "batch stream");
            cudaEventCreateWithFlags(&B.in[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&B.ran[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&B.out[i], cudaEventDisableTiming);
        }
    }
    if (!B.buf[0]) {
        for (int i = 0; i < 3; ++i)
            if ((e = cudaMalloc(&B.buf[i], bytes)) != cudaSuccess) {
                for (int j = 0; j < 3; ++j) {
                    cudaFree(B.buf[j]);
                    B.buf[j] = nullptr;
                }
                return cuda_status(e, "batch cudaMalloc");
            }
        B.bytes = bytes;
    }
    B.device = d;
    return SVB_OK;
}

int svb_host_run_ops_batch(const double *const *host_in, double *const *host_out, int nbatch,
                           int64_t n_amps, const svb_op *ops, int nops, unsigned flags) {
    if (nbatch < 0 || (nbatch > 0 && (!host_in || !host_out))) {
        set_error("batch: nbatch %d, host_in %p, host_out %p", nbatch, (const void *)host_in, (const void *)host_out);
        return SVB_EINVAL;
    }
    int r;
    for (int k = 0; k < nbatch; ++k) {
        if ((r = check_amps(host_in[k], n_amps)) != SVB_OK) return r;
        if ((r = check_amps(host_out[k], n_amps)) != SVB_OK) return r;
    }
    if ((r = check_ops(log2_exact(n_amps), ops, nops)) != SVB_OK) return r;
    if (nbatch == 0) return SVB_OK;
    std::lock_guard<std::mutex> lk(g_batch.mu);
    const size_t bytes = size_t(n_amps) * 16;
    if ((r = batch_setup(bytes)) != SVB_OK) return r;
    BatchStage &B = g_batch;
    cudaError_t e;
    // stage k uses buffer k % 3: H2D(k) waits for D2H(k-3) of that buffer;
    // the run waits for its H2D; the D2H waits for its run
    for (int k = 0; k < nbatch; ++k) {
        const int b = k % 3;
        if (k >= 3) cudaStreamWaitEvent(B.s[0], B.out[b], 0);
        if ((e = cudaMemcpyAsync(B.buf[b], host_in[k], bytes, cudaMemcpyHostToDevice, B.s[0])) != cudaSuccess)
            return cuda_status(e, "batch H2D");
        cudaEventRecord(B.in[b], B.s[0]);
        cudaStreamWaitEvent(B.s[1], B.in[b], 0);
        if ((r = svb_run_ops(B.buf[b], n_amps, ops, nops, flags, B.s[1])) != SVB_OK) return r;
        cudaEventRecord(B.ran[b], B.s[1]);
        cudaStreamWaitEvent(B.s[2], B.ran[b], 0);
        if ((e = cudaMemcpyAsync(host_out[k], B.buf[b], bytes, cudaMemcpyDeviceToHost, B.s[2])) != cudaSuccess)
            return cuda_status(e, "batch D2H");
        cudaEventRecord(B.out[b], B.s[2]);
    }
    if ((e = cudaStreamSynchronize(B.s[2])) != cudaSuccess) return cuda_status(e, "batch sync");
    return SVB_OK;
}

int svb_release_staging(void) {
    {
        std::lock_guard<std::mutex> lk(g_stage.mu);
        if (g_stage.ptr) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(g_stage.device);
            cudaFree(g_stage.ptr);
            cudaSetDevice(cur);
        }
        g_stage.ptr = nullptr;
        g_stage.bytes = 0;
    }
    std::lock_guard<std::mutex> lk(g_batch.mu);
    if (g_batch.device >= 0) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(g_batch.device);
        for (int i = 0; i < 3; ++i) {
            cudaFree(g_batch.buf[i]);
            g_batch.buf[i] = nullptr;
        }
        cudaSetDevice(cur);
        g_batch.bytes = 0;
    }
    return SVB_OK;
}

int svb_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaDeviceSynchronize();
    prof_drain();
    for (int c = 0; c < PROF_NCLASSES; ++c) g_prof_ms[c] = 0.0, g_prof_n[c] = 0, g_prof_bytes[c] = 0;
    g_prof_enabled = on != 0;
    return SVB_OK;
}

int svb_profile_read(int cls, int64_t *launches, double *total_ms, int64_t *alg_bytes) {
    if (cls < 0 || cls >= PROF_NCLASSES) {
        set_error("profile class %d out of range", cls);
        return SVB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(g_prof_mu);
    prof_drain();
    if (launches) *launches = g_prof_n[cls];
    if (total_ms) *total_ms = g_prof_ms[cls];
    if (alg_bytes) *alg_bytes = g_prof_bytes[cls];
    return SVB_OK;
}

const char *svb_profile_class_name(int cls) {
    static const char *names[PROF_NCLASSES] = {"k_pair_high", "k_pair_low", "k_diag", "k_tiny", "k_fused",
                                               "k_exchange", "k_norm", "kpass_jit", "k_dense", "k_signal",
                                               "k_swap_bits"};
    return (cls >= 0 && cls < PROF_NCLASSES) ? names[cls] : "";
}

}  // extern "C"

// ---- partitioned state -----------------------------------------------------

struct svb_dist {
    int n, k, p;
    int64_t L;
    std::vector<int> dev;
    std::vector<double2 *> slab;
    std::vector<cudaStream_t> stream;
    std::vector<cudaEvent_t> ev;
    std::vector<double *> scratch;
    int64_t exchanges = 0;
    std::vector<int64_t> peer_bytes;
};

namespace {

int set_dev(int d) {
    cudaError_t e = cudaSetDevice(d);
    return e == cudaSuccess ? SVB_OK : cuda_status(e, "cudaSetDevice");
}

// stream b waits for everything already queued on stream a
int order_after(svb_dist *d, int b, int a) {
    if (a == b) return SVB_OK;
    int r = set_dev(d->dev[a]);
    if (r) return r;
    cudaError_t e = cudaEventRecord(d->ev[a], d->stream[a]);
    if (e == cudaSuccess) {
        set_dev(d->dev[b]);
        e = cudaStreamWaitEvent(d->stream[b], d->ev[a], 0);
    }
    return e == cudaSuccess ? SVB_OK : cuda_status(e, "cross-rank ordering");
}

// Pairwise exchange on global bit gb among `mask`-selected ranks.
int dist_exchange(svb_dist *d, const Gate &g, int gb, int cbit, int rank_bit_req) {
    int64_t half = d->L >> 1;
    for (int r = 0; r < d->p; ++r) {
        int q = r ^ (1 << gb);
        if (r > q) continue;
        if (rank_bit_req >= 0 && !((r >> rank_bit_req) & 1)) continue;
        // both sides see each other's earlier work before touching the slabs
        int rc = order_after(d, r, q);
        if (!rc) rc = order_after(d, q, r);
        if (rc) return rc;
        // lower rank owns pairs j < L/2, upper rank j >= L/2
        if ((rc = set_dev(d->dev[r]))) return rc;
        prof_begin(d->stream[r]);
        LaunchInfo li = launch_pair_update(d->slab[r], d->slab[q], 0, half, g, cbit, d->stream[r]);
        prof_end(d->stream[r], li);
        g_launches += li.kernels;
        SVB_CHECK_LAUNCH("dist exchange (low)");
        if ((rc = set_dev(d->dev[q]))) return rc;
        prof_begin(d->stream[q]);
        li = launch_pair_update(d->slab[r], d->slab[q], half, d->L, g, cbit, d->stream[q]);
        prof_end(d->stream[q], li);
        g_launches += li.kernels;
        SVB_CHECK_LAUNCH("dist exchange (high)");
        // later work on either rank waits for both halves
        rc = order_after(d, r, q);
        if (!rc) rc = order_after(d, q, r);
        if (rc) return rc;
        int64_t moved = (cbit >= 0 ? half / 2 : half) * 16 * 2;  // read + write of partner amps
        d->peer_bytes[r] += moved;
        d->peer_bytes[q] += moved;
    }
    d->exchanges += 1;
    return SVB_OK;
}

}  // namespace

extern "C" {

int svb_dist_create(int n, int k, const int *devices, void *const *slabs, svb_dist **out) {
    if (!out || !devices || !slabs || n < 1 || n > 62 || k < 0 || k > n - 1 || k > 16) {
        set_error("bad arguments to svb_dist_create (n=%d, k=%d)", n, k);
        return SVB_EINVAL;
    }
    svb_dist *d = new svb_dist();
    d->n = n;
    d->k = k;
    d->p = 1 << k;
    d->L = int64_t(1) << (n - k);
    int cur = 0;
    cudaGetDevice(&cur);
    for (int r = 0; r < d->p; ++r) {
        if (!slabs[r] || reinterpret_cast<uintptr_t>(slabs[r]) % 16) {
            set_error("slab %d is NULL or misaligned", r);
            delete d;
            return SVB_EINVAL;
        }
        d->dev.push_back(devices[r]);
        d->slab.push_back((double2 *)slabs[r]);
    }
    d->peer_bytes.assign(d->p, 0);
    int rc = SVB_OK;
    for (int r = 0; r < d->p && !rc; ++r) {
        rc = set_dev(d->dev[r]);
        cudaStream_t s;
        cudaEvent_t e;
        double *sc;
        if (!rc && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) rc = SVB_ECUDA;
        if (!rc) d->stream.push_back(s);
        if (!rc && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) rc = SVB_ECUDA;
        if (!rc) d->ev.push_back(e);
        if (!rc && cudaMalloc((void **)&sc, sizeof(double) * norm_scratch_doubles()) != cudaSuccess)
            rc = SVB_ENOMEM;
        if (!rc) d->scratch.push_back(sc);
        // peer access for every partner on a different device
        for (int b = 0; b < d->k && !rc; ++b) {
            int peer = d->dev[r ^ (1 << b)];
            if (peer == d->dev[r]) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, d->dev[r], peer);
            if (!can) {
                set_error("device %d cannot access peer %d", d->dev[r], peer);
                rc = SVB_ESTATE;
                break;
            }
            cudaError_t pe = cudaDeviceEnablePeerAccess(peer, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) rc = cuda_status(pe, "peer access");
            cudaGetLastError();
        }
    }
    cudaSetDevice(cur);
    if (rc) {
        if (g_err[0] == 0) set_error("svb_dist_create failed");
        svb_dist_destroy(d);
        return rc;
    }
    *out = d;
    return SVB_OK;
}

int svb_dist_apply_1q(svb_dist *d, const double q[8], int target) {
    if (!d) return SVB_EINVAL;
    if (target < 0 || target >= d->n) {
        set_error("qubit %d out of range for n=%d", target, d->n);
        return SVB_EINVAL;
    }
    Gate g = make_gate(q);
    int boundary = d->n - d->k;
    if (target >= boundary) return dist_exchange(d, g, target - boundary, -1, -1);
    for (int r = 0; r < d->p; ++r) {  // engine.py:348-356, ranks concurrent
        int rc = set_dev(d->dev[r]);
        if (rc) return rc;
        prof_begin(d->stream[r]);
        LaunchInfo li = launch_gate(d->slab[r], d->L, g, target, -1, d->stream[r]);
        prof_end(d->stream[r], li);
        g_launches += li.kernels;
        SVB_CHECK_LAUNCH("dist local gate");
    }
    return SVB_OK;
}

int svb_dist_apply_c1q(svb_dist *d, const double q[8], int control, int target) {
    if (!d) return SVB_EINVAL;
    if (control < 0 || control >= d->n || target < 0 || target >= d->n || control == target) {
        set_error("bad control/target (%d, %d) for n=%d", control, target, d->n);
        return SVB_EINVAL;
    }
    Gate g = make_gate(q);
    int boundary = d->n - d->k;
    if (control >= boundary) {  // regime (iii): the control selects ranks
        int cb = control - boundary;
        if (target >= boundary) return dist_exchange(d, g, target - boundary, -1, cb);
        for (int r = 0; r < d->p; ++r) {
            if (!((r >> cb) & 1)) continue;
            int rc = set_dev(d->dev[r]);
            if (rc) return rc;
            prof_begin(d->stream[r]);
            LaunchInfo li = launch_gate(d->slab[r], d->L, g, target, -1, d->stream[r]);
            prof_end(d->stream[r], li);
            g_launches += li.kernels;
            SVB_CHECK_LAUNCH("dist rank-controlled gate");
        }
        return SVB_OK;
    }
    if (target >= boundary)  // regime (ii): exchange restricted to bit-c set
        return dist_exchange(d, g, target - boundary, control, -1);
    for (int r = 0; r < d->p; ++r) {  // regime (i)
        int rc = set_dev(d->dev[r]);
        if (rc) return rc;
        prof_begin(d->stream[r]);
        LaunchInfo li = launch_gate(d->slab[r], d->L, g, target, control, d->stream[r]);
        prof_end(d->stream[r], li);
        g_launches += li.kernels;
        SVB_CHECK_LAUNCH("dist controlled gate");
    }
    return SVB_OK;
}

int svb_dist_norm2(svb_dist *d, double *out) {
    if (!d || !out) return SVB_EINVAL;
    double total = 0.0;
    for (int r = 0; r < d->p; ++r) {
        int rc = set_dev(d->dev[r]);
        if (rc) return rc;
        g_launches += launch_norm2(d->slab[r], d->L, d->scratch[r], d->stream[r]);
        double v = 0.0;
        cudaError_t e = cudaMemcpyAsync(&v, d->scratch[r] + norm_scratch_doubles() - 1,
                                        sizeof(double), cudaMemcpyDeviceToHost, d->stream[r]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream[r]);
        if (e != cudaSuccess) return cuda_status(e, "svb_dist_norm2");
        total += v;  // rank order, like engine.py:453-454
    }
    *out = total;
    return SVB_OK;
}

int svb_dist_stats(svb_dist *d, int64_t *exchanges, int64_t *peer_bytes_per_rank) {
    if (!d) return SVB_EINVAL;
    if (exchanges) *exchanges = d->exchanges;
    if (peer_bytes_per_rank)
        for (int r = 0; r < d->p; ++r) peer_bytes_per_rank[r] = d->peer_bytes[r];
    return SVB_OK;
}

int svb_dist_sync(svb_dist *d) {
    if (!d) return SVB_EINVAL;
    for (int r = 0; r < d->p; ++r) {
        set_dev(d->dev[r]);
        cudaError_t e = cudaStreamSynchronize(d->stream[r]);
        if (e != cudaSuccess) return cuda_status(e, "svb_dist_sync");
    }
    return SVB_OK;
}

int svb_dist_destroy(svb_dist *d) {
    if (!d) return SVB_OK;
    for (size_t r = 0; r < d->stream.size(); ++r) {
        cudaSetDevice(d->dev[r]);
        cudaStreamSynchronize(d->stream[r]);
        cudaStreamDestroy(d->stream[r]);
    }
    for (size_t r = 0; r < d->ev.size(); ++r) {
        cudaSetDevice(d->dev[r]);
        cudaEventDestroy(d->ev[r]);
    }
    for (size_t r = 0; r < d->scratch.size(); ++r) {
        cudaSetDevice(d->dev[r]);
        cudaFree(d->scratch[r]);
    }
    delete d;
    return SVB_OK;
}

}  // extern "C"
