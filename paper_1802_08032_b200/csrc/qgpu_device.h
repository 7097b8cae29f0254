// qgpu_device.h — data layout and kernel-parameter structs shared by the
// host runtime (runtime.cpp) and the sm_100a kernels (kernels.cu).
//
// Amplitudes live in HBM as interleaved complex doubles (double2), the same
// bytes as the reference's std::complex<double> AmpVector
// (/root/reference/proj/include/qsim/register.hpp:13-42): qubit q contributes
// 2^q to an index (LSB = qubit 0), and a density matrix rho_jk sits at flat
// index j + 2^N k (register.hpp:47-50).
#pragma once

#include <cstdint>

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
// A CTA owns a tile of 2^kTileQubits amplitudes: the 5 lowest qubits (the
// lanes: every warp access is 512 contiguous bytes) plus kTileHigh arbitrary
// higher qubits. The ops of a pass run in phases; in each phase every thread
// holds 2^kPhaseRegBits amplitudes in registers spanning 4 of the tile's high
// qubits (the phase's register qubits), the 8 warps span the other 3. Gates
// on lane qubits use warp shuffles, gates on register qubits stay in
// registers, diagonal ops and channels act elementwise anywhere; between
// phases the tile is re-laid out through shared memory. Phase 0 loads from
// HBM and the last phase stores to HBM, so a pass is one read + one write of
// the state whatever its op count.
constexpr int kTileQubits = 12;
constexpr int kTileHigh = kTileQubits - kLaneQubits; // 7
constexpr int kPhaseRegBits = 4;
constexpr int kTileWarpBits = kTileHigh - kPhaseRegBits; // 3
constexpr int kTileThreads = 32 << kTileWarpBits;        // 256
constexpr int kMaxPhases = 8;
constexpr int kMaxTileOps = 64;

enum TileLoc : uint8_t { TL_LANE = 0, TL_REG = 1, TL_WARP = 2, TL_OUTER = 3 };

struct TileOp {
    uint8_t kind;    // PassOpKind (PO_PAIR_REG / PO_PAIR_LANE / PO_DIAG / ...)
    uint8_t cls;     // GateClass
    uint8_t flags;   // DiagFlags / collapse two-qubit flag
    uint8_t outcome;
    uint8_t q0k, q0p, q1k, q1p; // TileLoc kind + position of the op's qubits
    uint8_t lane_cmask;   // controls on lane bits
    uint8_t reg_cmask;    // controls on register-index bits
    uint8_t warp_cmask;   // controls on warp-index bits
    uint8_t pad[5];
    uint64_t outer_cmask; // controls on qubits outside the tile (global bits)
    double m[8];
};
static_assert(sizeof(TileOp) == 88, "TileOp layout");

struct TilePhase {
    uint16_t reg_off[1 << kPhaseRegBits];  // tile index of register i (lane 0, warp 0)
    uint16_t warp_off[1 << kTileWarpBits]; // tile index offset of warp w
    uint16_t op_begin, op_end;
};

struct TileParams {
    uint64_t num_tiles;
    uint64_t global_offset;
    int32_t num_phases;
    int32_t high_pos[kTileHigh];           // ascending global qubits of tile bits 5..
    uint64_t seg_off[1 << kTileHigh];      // global offset of tile segment s
    TilePhase phases[kMaxPhases];
    TileOp ops[kMaxTileOps];
};

} // namespace qgpu
