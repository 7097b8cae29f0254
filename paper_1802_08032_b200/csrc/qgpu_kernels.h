// qgpu_kernels.h — host-side launchers for the sm_100a kernels in kernels.cu.
// Every launcher enqueues on the given stream and returns immediately.
#pragma once

#include "qgpu_device.h"

#include <cuda_runtime.h>
#include <cstdint>

namespace qgpu {

// Number of reduction partials a reduce launch writes (fixed grid => the
// summation order, and so the result, is independent of timing).
constexpr int kReduceBlocks = 592; // 4 x 148 SMs
constexpr int kReduceThreads = 256;

// Kernel launches issued by this library since load (the bench's
// gpu_launches and the tests' evidence that the CUDA path ran).
uint64_t launch_count();
void count_launch(); // internal: every launcher calls it once per kernel

// Fused pass: applies params.ops in order to every amplitude in one HBM
// read + write (kernels.cu: k_fused_pass).
void launch_pass(double2* amps, const PassParams& params, cudaStream_t s);

// Tile pass (tile_pass.cu: k_tile_pass): 2^12-amplitude tiles streamed through
// shared memory by TMA, ops applied in register phases; one HBM read + write
// per pass.
void launch_tile_pass(void* amps, const TileParams& params, cudaStream_t s); // double2 or float2 (params.single)

// Per-pass JIT (tile_jit.cpp): launches the compiled kernel for this pass
// shape and returns true, or returns false (not compiled yet / JIT off).
bool launch_tile_pass_jit(void* amps, const TileParams& params, cudaStream_t s);
void jit_wait();              // block until every queued compile finished
void jit_set_mode(int mode);  // 0 off, 1 background compiles, 2 compile before first use
int jit_mode();
void jit_shutdown();
void jit_stats(unsigned long long* kernels, unsigned long long* failed, unsigned long long* pending);
int jit_selftest(char* log, int len, double* seconds); // host only: cubin bytes or -1

// The launchers below take type-erased amplitude pointers: `single` selects
// the float2 (Precision::Single) instantiation, else double2.

// One 2x2 gate over all pairs (i, i + 2^t) whose base holds cmask
// (reference kernels.cpp:43-59). Used for states too small to tile and for
// the unfused (one pass per gate) mode.
void launch_gate_simple(void* amps, bool single, int local_qubits, int target,
                        uint64_t cmask, const Mat2& m, int cls, cudaStream_t s);

// Elementwise ops on a contiguous range [0, len) whose global index of
// element 0 is goff (qubits are global qubit numbers).
void launch_diag_simple(void* amps, bool single, uint64_t len, uint64_t goff, int target,
                        uint64_t cmask, const Mat2& m, uint8_t flags, cudaStream_t s);
void launch_dephase(void* amps, bool single, uint64_t len, uint64_t goff, int q0, int q1,
                    double scale, cudaStream_t s);
void launch_collapse(void* amps, bool single, uint64_t len, uint64_t goff, int q0, int q1,
                     int outcome, double scale, cudaStream_t s);

// Depolarising 4-groups with both qubits local (density.cpp:62-81).
void launch_depolarise(void* amps, bool single, int local_qubits, int t, int tN,
                       double keep, double swap, double off, cudaStream_t s);

// Exchange combine (distributed.cpp:174-187): mine[i] <- own_lo ?
// lo_out(mine, theirs) : hi_out(theirs, mine) for local index idx0 + i whose
// bits hold low_mask.
void launch_combine(void* mine, const void* theirs, bool single, uint64_t len,
                    uint64_t idx0, uint64_t low_mask, int own_lo, const Mat2& m,
                    int cls, cudaStream_t s);

// Depolarising with the bra qubit on the rank bits: own_col = this rank's
// value of that bit; partner element of local index i is theirs[i ^ 2^t].
void launch_combine_depol(void* mine, const void* theirs, bool single, uint64_t len,
                          uint64_t idx0, int t, int own_col, double keep,
                          double swap, double off, cudaStream_t s);

// Compensated reductions (double-double accumulation in either precision).
// result = (hi, lo) double-double on the device.
// reduce_norm: sum |a_i|^2 over i in [0, len) (global index goff + i) with
// bit t == outcome (t < 0: all).
void launch_reduce_norm(const void* amps, bool single, uint64_t len, uint64_t goff, int t,
                        int outcome, double2* partials, double2* result,
                        cudaStream_t s);
// reduce_diag: sum Re (comp 0) or Im (comp 1) rho_jj over diagonal elements held in this range
// (flat index j (2^N + 1) in [goff, goff + len)) with bit t of j == outcome.
void launch_reduce_diag(const void* amps, bool single, uint64_t len, uint64_t goff, int N,
                        int t, int outcome, int comp, double2* partials,
                        double2* result, cudaStream_t s);

// every amplitude = re + i im (narrowed to float for single)
void launch_fill(void* amps, bool single, uint64_t len, double re, double im, cudaStream_t s);

} // namespace qgpu
