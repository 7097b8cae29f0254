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
// Host<->device bytes since load: explicit copies plus the op tables the
// pass kernels receive as launch parameters (TileParams / PassParams).
void count_transfer(uint64_t h2d, uint64_t d2h);
void transfer_bytes(uint64_t* h2d, uint64_t* d2h);

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
// writes pass k's generated program (both coefficient variants) to
// dir/pass_<k>.cu and dir/pass_<k>_smem.cu (dry runs, offline inspection)
void jit_dump_program(const TileParams& P, const char* dir, int k);
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

// Peer-memory exchange (single-node transport, peer.h): one rank updates
// both members of each pair, its own element and its partner's through a
// mapped peer pointer; the pair's two ranks take halves of the range.
// Exchange gate on local indices [begin, begin + n): (lo_side[i], hi_side[i])
// <- G (lo_side[i], hi_side[i]) where (i & low_mask) == low_mask.
void launch_peer_combine(void* lo_side, void* hi_side, bool single, uint64_t begin, uint64_t n,
                         uint64_t low_mask, const Mat2& m, int cls, cudaStream_t s);
// Qubit swap: elements [e0, e0 + n) of the traded half space, own side has
// bit v == side_own, the remote side the other value; exchanged in place.
void launch_peer_swap(void* own, void* remote, bool single, uint64_t e0, uint64_t n, int v, int side_own,
                      cudaStream_t s);
// Depolarising corner pairs [k0, k0 + n) between the rank whose bra bit is 0
// (col0) and its partner (col1), t = the ket qubit's local position.
void launch_peer_combine_depol(void* col0, void* col1, bool single, uint64_t k0, uint64_t n, int t,
                               double keep, double swap, cudaStream_t s);
// amps[i] *= f where bit t of local index i == bit
void launch_scale_bit(void* amps, bool single, uint64_t len, int t, int bit, double f, cudaStream_t s);

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

// All single-qubit marginals of a state-vector partition of 2^m amplitudes
// (m >= 13) in one read: out[0] = sum |a|^2, out[1 + q] = the sum over
// local index bit q == 1 (double-double, deterministic). `scratch` holds
// marginals_scratch_bytes(m).
constexpr int kMarginalsMinQubits = 13;
size_t marginals_scratch_bytes(int m);
void launch_marginals(const void* amps, bool single, int m, void* scratch, double2* out, cudaStream_t s);
// sum |a|^2 over the local indices i with (i & mask) == val (popcount(mask)
// <= 8): reads only the selected amplitudes
void launch_reduce_norm_sel(const void* amps, bool single, uint64_t len, uint64_t mask, uint64_t val,
                            double2* partials, double2* result, cudaStream_t s);

// every amplitude = re + i im (narrowed to float for single)
void launch_fill(void* amps, bool single, uint64_t len, double re, double im, cudaStream_t s);

} // namespace qgpu
