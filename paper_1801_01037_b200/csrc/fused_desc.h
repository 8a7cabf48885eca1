// fused_desc.h -- fused-pass descriptor layout shared by the interpreter
// kernel (fused.cu) and the runtime-specialised kernels (jit.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace svb {

#ifndef SVB_FM
#define SVB_FM 11
#endif
constexpr int FM = SVB_FM;             // qubits per tile
constexpr int FTILE = 1 << FM;         // 2048 amplitudes = 32 KiB
#ifndef SVB_FSLOTS
#define SVB_FSLOTS 4
#endif
constexpr int FSLOTS = SVB_FSLOTS;     // register bits per thread
constexpr int FREGS = 1 << FSLOTS;     // 16 amplitudes per thread
constexpr int FTHREADS = FTILE / FREGS;  // 128 threads
constexpr int FTBITS = FM - FSLOTS;    // 7 thread bits
// Tiles of runtime-specialised (JIT) passes may be larger than the
// interpreter's, with more amplitudes per thread: descriptors carry their own
// fm (11..FMMAX qubits) and fs (slot bits, 4..FSMAX)
constexpr int FMMAX = 13;
constexpr int FSMAX = 5;
constexpr int FREGMAX = 1 << FSMAX;
constexpr int FTBMAX = FMMAX - 4;  // thread bits at the largest tile, 4 slots
constexpr int FMAXG = 192;             // gates per pass
constexpr int FMAXGRP = 64;            // register groups per pass
constexpr int FMAXROWS = FTILE / 8;    // rows when flow = 3
#ifndef SVB_FCTAS
#define SVB_FCTAS 4
#endif
constexpr int FCTAS_PER_SM = SVB_FCTAS;
#ifndef SVB_FUSE_DB
#define SVB_FUSE_DB 0
#endif
constexpr bool kDB = SVB_FUSE_DB != 0;  // double-buffered tiles (next tile prefetched)
constexpr int kNBuf = kDB ? 2 : 1;
// default: 4 CTAs x (32 KiB tile + 2 KiB row table), 4 x 128 threads x 128 registers

// Opcodes (slot strides FSMAX whatever the pass's fs).  Non-diagonal:
// op = (kind * FSMAX + tslot) * 2 + ctrl.  Diagonal: FOP_DIAG + (var *
// (FSMAX + 1) + tpos) * 2 + ctrl, tpos = FSMAX meaning the target is a thread
// bit (one factor for all registers).
// ctrl = 1: a control on a slot, applied through the register mask cmask; a
// control on a thread bit is the per-thread predicate `cl`.
enum FKind { FK_GENERAL = 0, FK_REAL, FK_ANTI, FK_RX, FK_UANTI, FK_X, FK_Y, FK_NKIND };
enum FDiag { FD_GENERAL = 0, FD_D1, FD_Z, FD_S, FD_SDG, FD_NVAR };
constexpr int FOP_DIAG = FK_NKIND * FSMAX * 2;
constexpr int FTPOS_THREAD = FSMAX;  // diagonal tpos: target on a thread bit
// FGate.cl / FGate.tl >= FTILEBIT: the qubit lies outside the tile, at
// tile-index bit (value - FTILEBIT) -- a predicate uniform over the tile
// (runtime-specialised passes only; the interpreter never gets one)
constexpr int FTILEBIT = 64;

struct FGate {
    double2 m[4];
    uint8_t op;
    int8_t tl;       // diag with a thread-bit target: its thread bit (>= FTILEBIT: tile bit)
    int8_t cl;       // control on a thread bit: its thread bit (>= FTILEBIT: tile bit), else -1
    uint8_t u;       // FK_UANTI unit codes: bits 0-1 q12, bits 2-3 q21
    uint32_t cmask;  // ctrl = 1: registers (pairs: lo registers) the control allows
};
struct FGroup {
    int8_t pos[FSMAX];   // slot -> local bit
    int8_t tmap[FTBMAX]; // thread bit -> local bit
    int16_t first, count;
    // X / CNOT gates of the group, as the affine bit map P(l) = M l ^ mb they
    // induce on local indices: applied for free by storing register l at P(l)
    int16_t mb;
    int16_t mcol[FMMAX]; // column j of M = P(e_j) ^ mb
    int16_t perm;        // P is not the identity
    // byte offsets in the swizzled tile (host-precomputed, XOR-combined):
    int16_t qb, qcol[FMMAX];                        // load map Q (leading X / CNOT)
    uint32_t ld_b, ld_t[FTBMAX], ld_s[FSMAX];       // load through Q: offset, thread bits, slots
    uint32_t st_b, st_t[FTBMAX], st_s[FSMAX];       // store through P
};
struct FPass {
    int ngates, ngroups, ncomp, flow;
    int fm;                         // tile qubits (== FM for the interpreter)
    int fs;                         // slot bits per thread (== FSLOTS for the interpreter)
    int direct_first, direct_last;  // first/last group move registers <-> HBM directly
    int64_t gl_b, gl_t[FTBMAX], gl_s[FSMAX];         // first group: offsets through its load map
    int64_t gs_b, gs_t[FTBMAX], gs_s[FSMAX];         // last group: offsets through its store map
    int8_t comp[64];      // tile-index bit j -> global qubit comp[j]
    int8_t rowbit[FMMAX]; // local bit flow+j -> global qubit rowbit[j]
    FGroup groups[FMAXGRP];
    FGate gates[FMAXG];
};
static_assert(sizeof(FPass) <= 32000, "FPass is a __grid_constant__ kernel parameter");

}  // namespace svb
