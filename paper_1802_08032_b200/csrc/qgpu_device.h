// qgpu_device.h — data layout and kernel-parameter structs shared by the
// host runtime (runtime.cpp) and the sm_100a kernels (kernels.cu).
//
// Amplitudes live in HBM as interleaved complex doubles (double2), the same
// bytes as the reference's std::complex<double> AmpVector
// (/root/reference/proj/include/qsim/register.hpp:13-42): qubit q contributes
// 2^q to an index (LSB = qubit 0), and a density matrix rho_jk sits at flat
// index j + 2^N k (register.hpp:47-50).
#pragma once

#ifdef __CUDACC_RTC__ // NVRTC (tile_jit.cpp): no host headers
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef long long int64_t;
#else
#include <cstdint>
#endif

namespace qgpu {

// Lanes of a warp always span qubits 0..4: every warp-wide load/store moves
// 32 consecutive amplitudes = 512 contiguous bytes.
constexpr int kLaneQubits = 5;
constexpr int kMaxRegQubits = 5;   // per-thread register tile: 2^H amplitudes
constexpr int kMaxPassOps = 48;    // ops fused into one HBM pass

// Gate "class" = exact-zero pattern of the 2x2 matrix. Every class computes
// the reference's contracted fma chain (pair_math.hpp:30-45, see
// qsim_oracle.c) with the terms whose coefficient is exactly zero dropped;
// dropping an fma with a zero factor adds a signed zero, so every class is
// value-identical to the reference.
enum GateClass : uint8_t {
    CLS_GENERIC = 0, // no structure assumed
    CLS_REAL = 1,    // all imaginary parts zero (H, Ry, real rotations)
    CLS_RX = 2,      // a_im = b_re = c_re = d_im = 0 (Rx family)
    CLS_SWAP = 3,    // exactly [[0,1],[1,0]] (X / CNOT): a pure swap
    CLS_DIAG = 4,    // b = c = 0: elementwise phase (Z, S, T, Rz, CPhase)
};

// Where a qubit lives inside a fused pass.
enum LocKind : uint8_t { LOC_LANE = 0, LOC_REG = 1, LOC_OUTER = 2 };

struct QubitLoc {
    uint8_t kind; // LocKind
    uint8_t pos;  // lane bit, register-index bit, or global qubit
};

enum PassOpKind : uint8_t {
    PO_PAIR_REG = 0,  // 2x2 gate, target = register bit
    PO_PAIR_LANE = 1, // 2x2 gate, target = lane bit (warp shuffle)
    PO_DIAG = 2,      // diagonal gate, elementwise (any location)
    PO_DEPHASE = 3,   // scale where bit(q0) != bit(q1)
    PO_COLLAPSE = 4,  // keep where bit(q0) (and bit(q1)) == outcome, scale
};

enum DiagFlags : uint8_t { DF_A_ONE = 1, DF_D_ONE = 2 };

struct PassOp {
    uint8_t kind;     // PassOpKind
    uint8_t cls;      // GateClass (pair ops)
    uint8_t flags;    // DiagFlags / collapse: bit0 = two-qubit (density)
    uint8_t outcome;  // collapse outcome
    QubitLoc q0, q1;  // target (and partner qubit for channels)
    uint32_t lane_cmask;  // control bits among lane qubits
    uint32_t reg_cmask;   // control bits among register-index bits
    uint64_t outer_cmask; // control bits among the remaining (global) qubits
    double m[8];          // a_re a_im b_re b_im c_re c_im d_re d_im / scale
};
static_assert(sizeof(PassOp) == 88, "PassOp layout");

struct PassParams {
    uint64_t num_tiles;     // warp tiles: 2^(local_qubits - 5 - H)
    uint64_t global_offset; // global index of local amplitude 0 (rank offset)
    int32_t H;              // register qubits
    int32_t num_ops;
    int32_t reg_pos[kMaxRegQubits]; // ascending local qubit positions
    int32_t pad;
    uint64_t reg_off[1 << kMaxRegQubits]; // deposit(i, reg_pos)
    PassOp ops[kMaxPassOps];
};

struct Mat2 {
    double m[8];
};

// ------------------------------------------------------------ tile pass
//
// A CTA owns tiles of 2^kTileQubits amplitudes: the 5 lowest qubits (the
// lanes: every warp access is 512 contiguous bytes) plus kTileHigh arbitrary
// higher qubits. Its 16 warps form two tile groups of 8 that work on
// alternate tiles, so one group's phase transitions (shared-memory round
// trips and barriers) overlap the other group's arithmetic. The ops of a
// pass run in phases; in each phase every thread of a group holds
// 2^kPhaseRegBits = 16 amplitudes in registers spanning 4 of the tile's
// qubits (the phase's register qubits), 2 more ride on lane bits 3-4 and the
// 8 warps span the remaining 3. Measured on the 30-qubit bench circuit
// against one group of 16 warps with 8 register amplitudes (3 register
// qubits): 4 % faster end to end (profiles/r2_tile_groups.md) — most passes
// need two phases instead of three. Gates on lane qubits use warp shuffles,
// gates on register qubits stay in registers, diagonal ops and channels act
// elementwise anywhere; between phases the tile is re-laid out through
// shared memory. Phase 0 loads from HBM (TMA) and the last phase stores to
// HBM, so a pass is one read + one write of the state whatever its op count.
#ifndef QGPU_PHASE_REG_BITS
#define QGPU_PHASE_REG_BITS 4
#endif
#ifndef QGPU_TILE_GROUP_BITS
#define QGPU_TILE_GROUP_BITS 1
#endif
#ifndef QGPU_TILE_WARP_BITS
#define QGPU_TILE_WARP_BITS (4 - QGPU_TILE_GROUP_BITS)
#endif
constexpr int kPhaseRegBits = QGPU_PHASE_REG_BITS;
constexpr int kTileWarpBits = QGPU_TILE_WARP_BITS;  // warps per tile group: 2^WB
constexpr int kTileGroupBits = QGPU_TILE_GROUP_BITS; // independent tile groups per CTA
constexpr int kTileQubits = kLaneQubits + kPhaseRegBits + kTileWarpBits;
constexpr int kTileHigh = kTileQubits - kLaneQubits;
constexpr int kTileThreads = 32 << (kTileWarpBits + kTileGroupBits); // 512 (16 warps)
// Named barriers (IDs 1..15) of the phase transitions: one CTA-wide group
// uses them all (its full barrier is __syncthreads, ID 0); with two groups
// each owns seven, the first being its full-group barrier.
constexpr int kTileGroups = 1 << kTileGroupBits;
// QGPU_TILE_LDG=1: phase 0 reads HBM straight into registers (coalesced
// 16-byte loads of tiles prefetched into L2 by cp.async.bulk.prefetch) instead
// of TMA copies into shared memory; shared memory then only carries the
// phase transitions (one tile buffer per group), and a one-phase pass does
// not touch it at all.
#ifndef QGPU_TILE_LDG
#define QGPU_TILE_LDG 0
#endif
constexpr bool kTileLdg = QGPU_TILE_LDG != 0;
constexpr int kTileStages = kTileLdg ? (1 << QGPU_TILE_GROUP_BITS) : 3; // shared-memory tile buffers
constexpr int kTilePrefetch = 2; // LDG mode: tiles per group prefetched into L2 ahead
constexpr int kBarIdsPerGroup = kTileGroups == 1 ? 16 : 15 / kTileGroups; // relative IDs [1, this)
constexpr int kBarGroupBase = kTileGroups == 1 ? 0 : 1; // group g's ID 0 = kBarGroupBase + g * kBarIdsPerGroup
// Resident tile-pass CTAs per SM: single precision holds its 8 register
// amplitudes in 16 registers, so two CTAs (64 registers per thread, 2 x 96 KiB
// of stages) fit and double the warps that hide shared-memory latency.
constexpr int kTileCtasF64 = 1, kTileCtasF32 = 2;
constexpr int kMaxPhases = 8;
constexpr int kMaxTileOps = 63; // + the stop bit of a phase fits a 64-bit op mask

enum TileLoc : uint8_t { TL_LANE = 0, TL_REG = 1, TL_WARP = 2, TL_OUTER = 3 };

// Handler codes of the tile pass, resolved on the host so the kernel
// dispatches each op with one jump table (tile_pass.cu: apply). "SEL" codes
// carry controls on lane or register qubits (a per-element predicate);
// controls on warp or outer qubits are uniform per warp and skip the op.
enum TileCode : uint8_t {
    // register-bit handlers take the bit from the header (q0 pos; q1 pos for
    // the second qubit of a channel), a literal in JIT programs
    TC_REG = 0,      // + {GENERIC, REAL, RX, SWAP}: 0..3
    TC_REG_SEL = 4,  // + {GENERIC, SWAP}: 4..5
    TC_LANE_GENERIC = 6,
    TC_LANE_REAL = 7,
    TC_LANE_SWAP = 8,
    TC_LANE_SEL_GENERIC = 9,
    TC_LANE_SEL_SWAP = 10,
    TC_DIAG_REG = 11,       // both sides (Rz, diag(a, d))
    TC_DIAG_REG_D = 12,     // a == 1 (Z, S, T, phase shift)
    TC_DIAG_REG_SEL = 13,
    TC_DIAG_REG_D_SEL = 14,
    TC_DIAG_LANE = 15,      // target on a lane qubit
    TC_DIAG_LANE_SEL = 16,
    TC_DIAG_UNIFORM = 17,   // target on a warp / outer qubit
    TC_DIAG_UNIFORM_SEL = 18,
    TC_DEPHASE = 19,
    TC_COLLAPSE = 20,
    TC_DEPOL = 21,      // register bits q0 pos < q1 pos
    TC_DEPOL_LANE = 22, // t on lane bit q0 pos, t+N on register bit q1 pos
    TC_LANE_RX = 23,    // Rx-class 2x2 on a lane bit (tolerance mode only: TileParams.fast)
    TC_LANE_XCHG = 24,  // exchange lane bit q0 pos with register bit q1 pos (pure moves)
    TC_NUM_CODES = 25,
};

// Op header packed in one 64-bit word (one constant-bank load per op):
//   [0,6) TileCode  [6,10) flags  [10] outcome  [11,13) q0 TileLoc
//   [13,19) q0 pos  [19,21) q1 TileLoc  [21,27) q1 pos  [27,32) lane cmask
//   [32,37) register cmask  [40,48) unit coefficients (tolerance mode)
//   [48,52) warp cmask
struct TileOp {
    uint64_t hdr;
    uint64_t outer_cmask; // controls on qubits outside the tile (global bits)
    double m[8];
};
static_assert(sizeof(TileOp) == 80, "TileOp layout");

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define QGPU_HD __host__ __device__
#else
#define QGPU_HD
#endif

QGPU_HD constexpr uint64_t tile_hdr(uint32_t code, uint32_t flags, uint32_t outcome,
                            uint32_t q0k, uint32_t q0p, uint32_t q1k, uint32_t q1p,
                            uint32_t lane_cm, uint32_t reg_cm, uint32_t warp_cm) {
    return uint64_t(code & 63) | uint64_t(flags & 15) << 6 |
           uint64_t(outcome & 1) << 10 | uint64_t(q0k & 3) << 11 | uint64_t(q0p & 63) << 13 |
           uint64_t(q1k & 3) << 19 | uint64_t(q1p & 63) << 21 | uint64_t(lane_cm & 31) << 27 |
           uint64_t(reg_cm & 31) << 32 | uint64_t(warp_cm & 15) << 48;
}

// Lane bits 0-2 always span qubits 0-2 (a quarter-warp's 8 lanes read 128
// contiguous bytes: conflict-free LDS/STS.128 on the linear tile); lane bits
// 3 and 4 may carry any tile qubit per phase, so qubits 3 and 4 can be
// register qubits like the high ones.
constexpr int kFixedLaneBits = 3;

struct TilePhase {
    uint16_t reg_off[1 << kPhaseRegBits];  // tile index of register i (lane 0, warp 0)
    uint16_t warp_off[1 << kTileWarpBits]; // tile index offset of warp w
    uint16_t lane_off[2];                  // tile index offsets of lane bits 3, 4
    uint16_t op_begin, op_end;
    // warp bits shared with the previous phase at the same (top) positions:
    // the transition into this phase syncs groups of 2^(WB - sync_bits) warps
    // on named barriers bar_base + group (each transition its own IDs)
    uint16_t sync_bits;
    uint16_t bar_base;
    // Swizzled layouts (runtime.cpp: a middle phase holding qubits 0-2 in
    // registers). swz != 0: shared-memory positions are XORs of per-part
    // offsets — reading: reg_off[i] ^ warp_off[w] ^ lane_in[lane bits];
    // writing: reg_out[i] ^ warp_out[w] ^ lane_out[lane bits] — instead of
    // sums with lane bits 0-2 on tile bits 0-2.
    uint16_t swz;
    uint16_t lane_in[5], lane_out[5];
    uint16_t reg_out[1 << kPhaseRegBits];
    uint16_t warp_out[1 << kTileWarpBits];
};

struct TileParams {
    uint64_t num_tiles;
    uint64_t global_offset;
    // local qubits outside the tile that every op of the pass needs at 1
    // (common outer controls, outer diagonal targets with a == 1): only the
    // tiles with those bits set are visited; the others stay untouched in HBM
    uint64_t skip_ones;
    int32_t num_phases;
    int32_t fin_run;                       // a warp's segments come in HBM runs of 2^fin_run
    int32_t high_pos[kTileHigh];           // global qubits of tile bits 5.. (any order)
    int32_t high_sorted[kTileHigh];        // the same qubits, ascending
    int32_t any_outer;                     // some op has controls outside the tile
    int32_t single;                        // amplitudes are float2 (else double2)
    // tolerance-mode handlers (the reordering schedule, Env::order == 1):
    // lane ops without operand selects, Rx-class lane ops
    int32_t fast;
    uint64_t seg_off[1 << kTileHigh];      // global offset of tile segment s
    // the last phase stores straight to HBM: local-index offsets of its
    // register i, warp w and lane bits 3, 4 (lane bits 0-2: qubits 0-2)
    uint64_t fin_greg[1 << kPhaseRegBits];
    uint64_t fin_gwarp[1 << kTileWarpBits];
    uint64_t fin_glane[2];
    // phase 0 under QGPU_TILE_LDG loads straight from HBM: the same offsets
    // for the first phase's layout
    uint64_t first_greg[1 << kPhaseRegBits];
    uint64_t first_gwarp[1 << kTileWarpBits];
    uint64_t first_glane[2];
    // the 8 segments warp w owns in the last phase (its warp bits fixed)
    uint8_t fin_seg[1 << kTileWarpBits][1 << (kTileHigh - kTileWarpBits)];
    TilePhase phases[kMaxPhases];
    TileOp ops[kMaxTileOps];
};

} // namespace qgpu
