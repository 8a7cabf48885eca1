/*
 * svb.h -- C ABI of the B200 state-vector gate engine (libsvb.so).
 *
 * Drop-in boundary for the reference package `svsim` (read-only at
 * /root/reference/pkg).  Each entry point names the reference interface it
 * replaces.  Plain pointers and sizes only: amplitude buffers are interleaved
 * complex128 (re, im) -- numpy complex128 on the host, CUDA double2 on the
 * device.  Gates cross as `const double q[8]` = re/im of q11, q12, q21, q22
 * (svsim.core.Gate2x2, core.py:67-94).  Streams are `cudaStream_t` passed as
 * `void*` (NULL = legacy default stream).
 *
 * Conventions: qubit i <-> index bit 2^i (core.py:3-9).  Return 0 on success,
 * a negative SVB_E* code on failure; svb_last_error() gives the message of
 * the calling thread's last failure.  The host layer maps SVB_EINVAL ->
 * ValidationError, SVB_ENOMEM -> CapacityError, SVB_ESTATE ->
 * ContractViolation, SVB_ECUDA/SVB_ENCCL -> SvsimError (errors.py:9-32).
 *
 * Arithmetic: every pair update is (q11*lo + q12*hi, q21*lo + q22*hi) with
 * complex products (ac-bd, ad+bc) in round-to-nearest, no FMA -- the
 * reference's compiled kernel built with -ffp-contract=off
 * (_stride_cy.pyx:16-21, setup.py:46-48) -- so single-gate results are
 * bit-identical to it (zeros may differ in sign only).
 */
#ifndef SVB_H
#define SVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVB_OK 0
#define SVB_EINVAL (-1)  /* bad argument                  -> ValidationError   */
#define SVB_ENOMEM (-2)  /* allocation failed / too large -> CapacityError     */
#define SVB_ECUDA (-3)   /* CUDA runtime error            -> SvsimError        */
#define SVB_ENCCL (-4)   /* communication error           -> SvsimError        */
#define SVB_ESTATE (-5)  /* call not allowed in state     -> ContractViolation */

/* One circuit operation: svsim.core.GateOp (core.py:97-115).
 * kind 0 = single (control ignored), 1 = controlled. */
typedef struct svb_op {
    int32_t kind;
    int32_t target;
    int32_t control;
    int32_t reserved;
    double q[8];
} svb_op;

/* svb_run_ops flags */
#define SVB_RUN_FUSE 1u         /* plan multi-gate shared-memory passes        */
#define SVB_RUN_STRICT_ORDER 2u /* fuse only contiguous runs (bit-exact order) */
#define SVB_RUN_FMA 4u          /* fused passes may contract a*b+c and (with JIT) pull
                                   scalars out of 1-qubit gates; <= 1e-12 (not with STRICT) */
#define SVB_RUN_JIT 8u          /* compile each fused pass to straight-line code (NVRTC,
                                   cached per op list): 12-qubit tiles, X/CNOT as register
                                   renames; falls back to the interpreter without NVRTC */
#define SVB_RUN_JIT_ASYNC 16u   /* with SVB_RUN_JIT: a plan whose passes are not compiled
                                   yet runs on the interpreter while NVRTC compiles them on
                                   a background thread; later calls switch over.  Compiled
                                   cubins are also kept on disk (SVB_JIT_CACHE, default
                                   $XDG_CACHE_HOME/svb-jit or ~/.cache/svb-jit; "0" = off),
                                   keyed by source, options and NVRTC version */

int svb_abi_version(void);
const char *svb_last_error(void);
/* Kernels launched by this library since load (all entry points). */
int64_t svb_launch_count(void);

/* Launch profiler: while enabled, every gate/exchange launch is bracketed by
 * CUDA events on its own stream and aggregated per kernel class (0
 * k_pair_high, 1 k_pair_low, 2 k_diag, 3 k_tiny, 4 k_fused, 5 k_exchange,
 * 6 k_norm, 7 kpass_jit) with its algorithmic HBM bytes.  enable() resets the totals; read()
 * synchronises on the recorded events. */
int svb_profile_enable(int on);
int svb_profile_read(int cls, int64_t *launches, double *total_ms, int64_t *alg_bytes);
const char *svb_profile_class_name(int cls);

/* ---- device buffers, stream-ordered (asynchronous) ---------------------- */

/* Replaces svsim.kernel.apply_single (kernel/__init__.py:107-117) and the
 * backend entry _stride_cy.apply_single (_stride_cy.pyx:24-54). */
int svb_apply_1q(void *amps, int64_t n_amps, const double q[8], int target, void *stream);

/* Replaces svsim.kernel.apply_controlled (kernel/__init__.py:120-134) and
 * _stride_cy.apply_controlled (_stride_cy.pyx:57-90). */
int svb_apply_c1q(void *amps, int64_t n_amps, const double q[8], int control, int target,
                  void *stream);

/* Applies ops[0..nops) in order -- the per-op loop of run_circuit for one
 * rank (engine.py:483-494) -- optionally fusing gates into shared-memory
 * passes (flags).  Results agree with op-by-op application within 1e-12;
 * with SVB_RUN_STRICT_ORDER they are bit-identical. */
int svb_run_ops(void *amps, int64_t n_amps, const svb_op *ops, int nops, unsigned flags,
                void *stream);

/* Number of trailing ops (a multiple of 3, 0 if none) that form a SWAP network
 * of CNOT triples -- pairwise disjoint, each of the five lowest qubits swapped
 * with a higher one: the QFT's final qubit reversal (workloads.qft_circuit;
 * reference form core.py SWAP = 3 CNOTs) -- which svb_run_ops applies in one
 * in-place HBM pass (k_swap_bits) after the fused passes of the ops before it.
 * Host only. */
int svb_swap_suffix(int n_qubits, const svb_op *ops, int nops);

/* Number of HBM passes svb_run_ops would make for these ops, and (groups,
 * may be NULL) the total shared-memory register groups of the fused passes.
 * Planner only, no device work. */
int svb_plan_passes(int n_qubits, const svb_op *ops, int nops, unsigned flags, int *passes,
                    int *groups);

/* Host-only: plan the op list, generate the SVB_RUN_JIT source of every fused
 * pass and compile it with NVRTC (no device work).  *compiled = passes
 * compiled; SVB_ESTATE (message in svb_last_error) when NVRTC is missing or a
 * pass fails to compile. */
int svb_jit_check(int n_qubits, const svb_op *ops, int nops, unsigned flags, int *compiled);
/* Runtime-specialised pass counters since load: cubins read from the on-disk
 * cache, and NVRTC compiles. */
void svb_jit_counters(long *disk_hits, long *compiles);
/* Block until the background compiles SVB_RUN_JIT_ASYNC started have finished. */
void svb_jit_wait(void);

/* sum |a_j|^2 -> *out (host).  Synchronises `stream`.  Replaces norm2
 * (core.py:171-174) / _dist_norm2 for one slab (engine.py:453-454). */
int svb_norm2(const void *amps, int64_t n_amps, double *out, void *stream);

/* probs[j] = |a_j|^2 into a device buffer of n_amps doubles. */
int svb_probs(const void *amps, int64_t n_amps, double *probs, void *stream);

/* ---- dense verifier (oracle.py:81-176), n <= 12 ---------- */

#define SVB_MAX_DENSE_QUBITS 12 /* oracle.py:22 MAX_DENSE_QUBITS */
/* Write the 2^n x 2^n embedding of gate q on `target` (control = -1: none;
 * else only where bit `control` is set) into u (row-major complex128):
 * embed_single / embed_controlled (oracle.py:81-116), the same bits.
 * n > 12: SVB_ENOMEM (the reference's CapacityError). */
int svb_dense_embed(void *u, int n_qubits, const double q[8], int control, int target, void *stream);
/* y[row0 .. row0+nrows) = (U x)[rows], U row-major dim x dim: matvec /
 * matvec_partitioned's per-rank strip (oracle.py:122-176).  Each row is a
 * fixed-order sum, so any row partition gives the same bits. */
int svb_dense_matvec(const void *u, const void *x, void *y, int64_t dim, int64_t row0, int64_t nrows,
                     void *stream);

/* Own-row exchange update of the paper's single-amplitude protocol for one
 * received chunk (engine.py:241-254 scheme b, 257-272 chunked): for
 * j in [0, count): own[j] = own_is_low ? q11*own[j] + q12*other[j]
 *                                      : q21*other[j] + q22*own[j],
 * restricted to local indices (index_offset + j) with bit cbit set when
 * cbit >= 0 (engine.py:199-203). */
int svb_exchange_own_row(void *own, const void *other, int64_t count, const double q[8],
                         int own_is_low, int cbit, int64_t index_offset, void *stream);

/* Qubit relabeling, out of place: dst[p] = src[s] where bit j of p is bit
 * phys_to_logical[j] of s (svsim.layout.permute_state, layout.py:71-83). */
int svb_permute_qubits(const void *src, void *dst, int64_t n_amps, const int *phys_to_logical, int n,
                       void *stream);

/* Control-masked exchange (regime ii, engine.py:444-447: only indices with
 * the local control bit set travel).  Packed index p stands for local index
 * insert_bit(offset + p, cbit, 1).  pack: dst[p] = src[that index], p in
 * [0, count).  own_row_packed: own[that index] = own-row update with
 * other_packed[p]. */
int svb_pack_ctrl(const void *src, void *dst, int64_t count, int cbit, int64_t offset, void *stream);

/* Half-slab gather / scatter for swapping a global (rank) qubit with a local
 * one (dynamic layout): packed index p stands for local index
 * insert_bit(offset + p, bit, value).  pack: dst[p] = src[that index];
 * unpack: dst[that index] = src[p].  A swap of rank bit g with local bit l
 * sends the half with local bit l != the rank's bit g to the partner rank
 * (rank ^ (1 << g)) and unpacks the partner's half into the same positions:
 * 8 L bytes each way instead of 16 L per global gate. */
int svb_pack_half(const void *src, void *dst, int64_t count, int bit, int value, int64_t offset, void *stream);
int svb_unpack_half(void *dst, const void *src, int64_t count, int bit, int value, int64_t offset, void *stream);
int svb_exchange_own_row_packed(void *own, const void *other_packed, int64_t count, const double q[8],
                                int own_is_low, int cbit, int64_t offset, void *stream);

/* Both rows for amplitude pairs held in two slabs (lo_slab[j], hi_slab[j]),
 * j in [begin, end), masked by local bit cbit when cbit >= 0.  The fused
 * peer-memory form of a global-target exchange (one side may be a peer
 * device's memory).  Arithmetic identical to the own-row rule. */
int svb_pair_update(void *lo_slab, void *hi_slab, int64_t begin, int64_t end, const double q[8],
                    int cbit, void *stream);

/* Peer-memory transport of the multi-process engine (DistEngine(peer=True);
 * replaces the send/recv of engine.py:359-389 and its layout swaps): every
 * rank exports its slab (svb_ipc_handle, 64 opaque bytes shipped over the
 * control-plane process group), opens its partners' (svb_ipc_open), and a
 * global-target gate or a layout swap runs as one kernel per rank that
 * reads and writes the partner slab in place -- svb_pair_update above, and
 * svb_peer_swap_half: for j in [begin, end) swap a[ins(j, bit, va)] with
 * b[ins(j, bit, vb)] (ins: insert the value as bit `bit` of j). */
int svb_peer_swap_half(void *a, void *b, int64_t begin, int64_t end, int bit, int va, int vb, void *stream);
/* handle of the allocation holding dev_ptr, and dev_ptr's byte offset in it
 * (svb_ipc_open returns the allocation's base: add the offset) */
int svb_ipc_handle(const void *dev_ptr, unsigned char handle[64], int64_t *offset);
int svb_ipc_open(const unsigned char handle[64], void **dev_ptr);
int svb_ipc_close(void *dev_ptr);
/* Stream-ordered pairwise rank synchronisation for the peer transport (no
 * host barrier): svb_stream_signal stores `value` into a (peer) device word
 * with system-scope release after every earlier kernel of `stream`;
 * svb_stream_wait makes `stream` wait until the local word is >= value
 * (cuStreamWaitValue32, no SM occupied).  Each rank of a pair signals its
 * partner's word and waits on its own, before and after the pair kernel.
 * Replaces the per-gate synchronize + process-group barrier around
 * engine.py:359-389's exchange. */
int svb_stream_signal(void *flag, uint32_t value, void *stream);
int svb_stream_wait(void *flag, uint32_t value, void *stream);
/* SM-driven copy dst[i] = src[i] (n_amps x 16 B; either side may be peer
 * memory): the link-ceiling probe of the multi-GPU bench. */
int svb_peer_copy(void *dst, const void *src, int64_t n_amps, void *stream);
/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault): the copy-engine leg
 * of the same probe (cudaMemcpyPeerAsync when the two sides sit on
 * different GPUs). */
int svb_copy_async(void *dst, const void *src, int64_t bytes, void *stream);
/* Page-lock a caller-owned host array (cudaHostRegister; already registered
 * is not an error) / release it.  backend.py registers large svsim arrays
 * once and releases them when the array is garbage-collected. */
int svb_host_register(void *host, int64_t bytes);
int svb_host_unregister(void *host);

/* ---- host buffers, synchronous (the svsim kernel-backend contract) ------ */

/* Backend-module contract apply_single(amps, q11, q12, q21, q22, target,
 * mode, workers) (_stride_py.py:93-98; _stride_cy.pyx:24-25): in place on a
 * host complex128 array; mode/workers are accepted and ignored. */
int svb_host_apply_1q(double *host_amps, int64_t n_amps, const double q[8], int target);
/* (From 2^22 amplitudes the state streams through the device in 64 MiB
 * units on three streams -- H2D, kernel and D2H of different units overlap
 * -- and units a high control bit switches off are not copied.  Pin the
 * caller's array once with svb_host_register for full-duplex PCIe.) */
int svb_host_apply_c1q(double *host_amps, int64_t n_amps, const double q[8], int control,
                       int target);
/* Whole op list on host memory: H2D of host_in, svb_run_ops, D2H into
 * host_out (may equal host_in).  Synchronous.  The end-to-end public call. */
int svb_host_run_ops(const double *host_in, double *host_out, int64_t n_amps, const svb_op *ops,
                     int nops, unsigned flags);
/* The same op list over a batch of host states (serving: many inputs, one
 * circuit): state k is copied in (host_in[k]), run and copied out
 * (host_out[k]) exactly as svb_host_run_ops would, but the three stages of
 * consecutive states overlap -- H2D of k+1 and D2H of k-1 on their own
 * streams while k runs -- through three device buffers owned by the
 * library.  Synchronous: returns when every host_out[k] is written.  Pinned
 * host buffers are needed for the copies to overlap.  host_out[k] may equal
 * host_in[k]; results equal nbatch calls of svb_host_run_ops bit for bit. */
int svb_host_run_ops_batch(const double *const *host_in, double *const *host_out, int nbatch,
                           int64_t n_amps, const svb_op *ops, int nops, unsigned flags);
/* Free the device staging buffers the host-memory calls keep between calls
 * (one state for svb_host_*, three for the batch call); they are
 * reallocated on the next call. */
int svb_release_staging(void);

/* ---- partitioned state over 2^k ranks (engine.py DistState) ------------- */

typedef struct svb_dist svb_dist;

/* n qubits over 2^k ranks; rank r's slab of 2^(n-k) amplitudes lives at
 * slabs[r] on device devices[r] (ranks may share a device).  Peer access is
 * enabled between distinct devices.  Does not take ownership of slabs. */
int svb_dist_create(int n, int k, const int *devices, void *const *slabs, svb_dist **out);
/* needs_comm(t) ? pairwise exchange : local sweep (engine.py:488-492). */
int svb_dist_apply_1q(svb_dist *d, const double q[8], int target);
/* The three controlled regimes (engine.py:415-450). */
int svb_dist_apply_c1q(svb_dist *d, const double q[8], int control, int target);
int svb_dist_norm2(svb_dist *d, double *out);
/* Cumulative per-rank exchange accounting: amplitudes each rank read from
 * and wrote to its partner's slab (peer traffic), and exchanges performed. */
int svb_dist_stats(svb_dist *d, int64_t *exchanges, int64_t *peer_bytes_per_rank);
int svb_dist_sync(svb_dist *d);
int svb_dist_destroy(svb_dist *d);

#ifdef __cplusplus
}
#endif
#endif /* SVB_H */
