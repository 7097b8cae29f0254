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

} // namespace qgpu
