/*
 * qgpu.h — extensions of the C-ABI beyond QuEST's names (libqgpu.so).
 *
 * Everything here is plain C: pointers, sizes, integers. The reference has no
 * equivalent for most of these (they expose B200 execution control); where it
 * has one, it is cited (paths under /root/reference/proj).
 */
#ifndef QGPU_EXT_H
#define QGPU_EXT_H

#include "QuEST.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------------- errors */
/* Error classes mirror the reference's exception types (types.hpp:31-55). */
enum qgpuErrorCode {
    QGPU_OK = 0,
    QGPU_DOMAIN_ERROR = 1,   /* qsim::DomainError: invalid argument, no mutation */
    QGPU_RESOURCE_ERROR = 2, /* qsim::ResourceError: allocation, bytes named */
    QGPU_COMM_ERROR = 3,     /* qsim::CommError: transport failure, ranks named */
    QGPU_DEVICE_ERROR = 4    /* CUDA runtime failure */
};
typedef void (*qgpuErrorHandler)(const char* errMsg, const char* errFunc, int code,
                                 void* user);
/* Replaces the default recording handler (NULL restores it). */
void qgpuSetErrorHandler(qgpuErrorHandler handler, void* user);
/* Code of the last error on this thread (0 = none); copies its message. */
int qgpuGetLastError(char* buf, int len);
void qgpuClearError(void);

/* ------------------------------------------------------ execution control */
const char* qgpuVersion(void);
/* Kernel launches issued by the library since load. */
unsigned long long qgpuKernelLaunches(void);
/* Host<->device bytes since load: explicit copies (amplitude reads/writes,
 * reduction results) plus the op tables the pass kernels receive as launch
 * parameters. Either pointer may be NULL. */
void qgpuTransferBytes(unsigned long long* h2d, unsigned long long* d2h);
/* HBM passes / exchange rounds executed for this register. */
unsigned long long qgpuPassCount(Qureg qureg);
/* Launch every queued op of this register now (stream-ordered, async). */
void qgpuFlush(Qureg qureg);
/* Fusion policy for registers of this env: mode 0 = fused HBM passes
 * (default), 1 = one fused-pass launch per op, 2 = one simple per-gate kernel
 * per op (the unfused kernel family). maxOps <= 0 keeps the current value,
 * regQubits in [1,5] (<= 0 keeps). */
void qgpuSetFusion(QuESTEnv env, int mode, int maxOps, int regQubits);
/* The CUDA stream (cudaStream_t) all work of this env is enqueued on. */
void* qgpuGetStream(QuESTEnv env);
int qgpuGetDevice(QuESTEnv env);

/* Launch profiling: while on, every hot-kernel launch (fused pass, simple
 * gate, exchange round, depolarise, reduction) is bracketed by a CUDA event
 * pair on the env's stream. Stop syncs and returns the record count, filling
 * up to maxRecords durations (ms) and kinds (0 pass, 1 simple, 2 exchange,
 * 3 depolarise, 4 reduce). */
void qgpuProfileStart(QuESTEnv env);
int qgpuProfileStop(QuESTEnv env, double* ms, int* kinds, int maxRecords);
/* Per-record detail of the last profile window (same order as
 * qgpuProfileStop): fused tile passes carry ops | phases << 8 | (modelled
 * FP64 instructions per amplitude x 4) << 16. */
int qgpuProfileInfo(QuESTEnv env, int* info, int maxRecords);

/* ------------------------------------------------------------- precision */
/* Register(num_qubits, kind, precision) (register.hpp:53-54): precision 1 =
 * Precision::Single (float2 amplitudes, float arithmetic: Mat2<float> and
 * channel factors narrowed once, kernels.cpp:61-62, density.cpp:105-140),
 * 2 = Precision::Double (what createQureg / createDensityQureg make). The
 * host boundary stays double: reads widen, writes narrow (register.cpp:
 * 30-51); reductions accumulate in double. Single-precision registers of
 * fewer than 12 local qubits run one kernel per op. */
Qureg qgpuCreateQuregPrecision(int numQubits, QuESTEnv env, int density, int precision);
int qgpuGetPrecision(Qureg qureg); /* 1 or 2; -1 on error */

/* ------------------------------------------------------------ run_circuit */
/* One op of a circuit (96 bytes): kind 0 = a 2x2 gate `m` (re, im of m00,
 * m01, m10, m11) on `target` with controls `ctrlMask` (bit c = qubit c), as
 * apply_controlled_gate / apply_gate_to_density (kernels.cpp:105-112,
 * density.cpp:85-116); kind 1 = apply_dephasing(target, prob); kind 2 =
 * apply_depolarising(target, prob) (density.cpp:118-145). */
typedef struct {
    int kind;
    int target;
    unsigned long long ctrlMask;
    double m[8];
    double prob;
    double reserved;
} qgpuOp;
/* run_circuit (circuit.cpp:239-247) in one call: all ops are validated first
 * (an invalid one leaves the register untouched and reports which), then
 * queued in order — the same results as one call per op, without a C-ABI
 * crossing per gate. */
void qgpuRunCircuit(Qureg qureg, const qgpuOp* ops, int numOps);

/* --------------------------------------------------------- bulk state I/O */
/* Interleaved (re, im) doubles of flat amplitudes [start, start + num). */
void qgpuCopyStateToHost(Qureg qureg, long long int start, long long int num, double* out);
void qgpuCopyStateFromHost(Qureg qureg, long long int start, long long int num,
                           const double* in);
/* Any 2x2 matrix (not checked for unitarity, as the reference allows
 * untagged matrices, gates.hpp:9-11) on `target` with controls `ctrlMask`:
 * apply_controlled_gate (kernels.cpp:105-112) / apply_gate_to_density. */
void qgpuApplyMatrix(Qureg qureg, int target, unsigned long long ctrlMask, const double* m8);
/* Reference-named reductions: Register::norm_squared (register.cpp:62-75,
 * compensated) and trace (density.cpp:147-154). */
qreal qgpuNormSquared(Qureg qureg);
Complex qgpuTrace(Qureg qureg);

/* ------------------------------------------------------------ distributed */
/* 2^k virtual ranks on this one GPU, each holding its own chunk, exchanging
 * through the same sub-chunked protocol as NCCL ranks (a device-side
 * InProcessTransport, transport.hpp:33-62). numRanks must be a power of 2. */
QuESTEnv qgpuCreateLoopbackEnv(int numRanks);
/* One process per GPU over NCCL (loaded at run time: the libnccl.so.2
 * already in the process, else the system one). Rank 0 calls
 * qgpuGetNcclUniqueId and distributes the 128 bytes. */
int qgpuGetNcclUniqueId(char* out128);
QuESTEnv qgpuCreateNcclEnv(int rank, int numRanks, int device, const char* uniqueId128);
/* One process per GPU of one node over peer memory (the default multi-GPU
 * transport; replaces Transport / InProcessTransport, transport.hpp:18-62):
 * every rank maps every rank's partition (CUDA IPC over NVLink/NVSwitch);
 * an exchange gate, a depolarising channel on a global bra qubit or a
 * global<->local qubit swap is one kernel per rank that updates its half of
 * the amplitude pairs in both partitions in place (no staging buffer, no
 * send/recv). Rank 0 calls qgpuPeerUniqueId (it creates the group's
 * shared-memory control segment) and distributes the 128 bytes; every rank
 * then calls qgpuCreatePeerEnv. A rank that exits, aborts or stalls past
 * QGPU_PEER_TIMEOUT_S makes its partners' calls fail with
 * QGPU_COMM_ERROR instead of hanging. */
int qgpuPeerUniqueId(char* out128);
QuESTEnv qgpuCreatePeerEnv(int rank, int numRanks, int device, const char* id128);
/* Host-only self test of a peer group's control plane (no GPU): attach as
 * `rank`, run `rounds` checked all-gathers and barriers; exitAfter >= 0
 * makes this process exit mid-protocol at that round (failure-detection
 * tests). Returns 0, or QGPU_COMM_ERROR with the reason in
 * qgpuGetLastError. */
int qgpuPeerProbe(const char* id128, int rank, int numRanks, int rounds, int exitAfter);
/* Exchange sub-chunk size in amplitudes (power of two, default 2^24). */
void qgpuSetExchangeChunk(QuESTEnv env, long long int amps);
/* Global<->local qubit swaps (default on): a gate whose target is a global
 * (rank-bit) qubit first swaps that qubit with the least recently used local
 * one — each rank trades half its partition with its partner once — instead
 * of exchanging the whole partition for every such gate as the reference
 * does (distributed.cpp:167-231). Amplitudes are bit-identical either way;
 * 0 selects the reference's per-gate exchange. Registers of this env are
 * first returned to the identity qubit layout. */
void qgpuSetQubitSwaps(QuESTEnv env, int enable);

/* Op order inside the fused HBM passes. 1 (default): ops that commute (they
 * meet only on qubits both act on diagonally — controls, phases, dephasing,
 * collapse — or share no qubit) are scheduled out of circuit order into
 * fewer passes; amplitudes equal the reference's up to rounding (within
 * 1e-12 max-abs, tested at 30 qubits), not bit for bit. 0: circuit order,
 * bit-identical to the reference (kernels.cpp:105-112, fma chain included).
 * windowOps > 0 sets how many queued ops the scheduler looks ahead (default
 * 512). Queued ops of this env's registers are flushed first. Environment:
 * QGPU_ORDER=exact|reorder, QGPU_WINDOW=n. */
void qgpuSetOrdering(QuESTEnv env, int reorder, int windowOps);
int qgpuGetOrdering(QuESTEnv env);

/* The tile-pass scheduler alone (host only, no GPU): numOps physical ops on
 * a flatQubits-qubit local state (kinds: 0 gate with its 8-double matrix
 * (re, im row-major) in mats[8 i], 1 dephasing, 2 depolarising on (q0, q1),
 * 3 collapse), scheduled as a register of that size would with the given
 * ordering, window and phase limit. Writes, per executed op in execution
 * order, its input index, pass and phase; returns the number of passes, or
 * -1 on invalid input. */
int qgpuPlanPasses(int flatQubits, int numOps, const int* kinds, const int* q0, const int* q1,
                   const unsigned long long* cmasks, const double* mats, int reorder, int windowOps,
                   int maxPhases, int* orderOut, int* passOut, int* phaseOut);

/* The swap planner alone (host only, no GPU): for numOps ops on logical
 * flat qubits targets[k] (pairOps[k] != 0 for a 2x2 non-diagonal gate,
 * 0 for a diagonal op) on 2^rankLog2 ranks, the swaps the runtime performs:
 * swapsOut[3i..3i+2] = (op index, global position, local position).
 * Returns the number of swaps, or -1 on invalid input. */
int qgpuPlanSwaps(int flatQubits, int rankLog2, unsigned long long chunkAmps, int numOps,
                  const int* targets, const int* pairOps, int* swapsOut, int maxSwaps);

/* The distributed schedule alone (host only, no GPU): the ops of
 * qgpuPlanPasses on logical flat qubits of a register split over
 * 2^rankLog2 peer-transport ranks, run through the runtime's own queue —
 * reorder != 0: the light-cone drain (any op that can run with the local
 * qubits first, swaps only when nothing can) and the reordering window;
 * 0: circuit order. swapsOut[2i..2i+1] = (global position, local position)
 * of the i-th swap; *passesOut = tile passes. Returns the number of swaps,
 * or -1 on invalid input. */
int qgpuPlanDistributed(int flatQubits, int rankLog2, int numOps, const int* kinds, const int* q0, const int* q1,
                        const unsigned long long* cmasks, const double* mats, int reorder, int* passesOut,
                        int* swapsOut, int maxSwaps);

/* Messages / bytes this process's ranks sent for `qureg` (CommStats,
 * distributed.hpp:63-74); arrays of length numRanks (loopback) or 1. */
void qgpuCommStats(Qureg qureg, unsigned long long* messages, unsigned long long* bytes);

/* Pure host planner used by every transport (testable without a GPU).
 * For a gate on flat qubit `target` with controls `ctrlMask` on a
 * 2^flatQubits vector split over 2^rankLog2 ranks (distributed.cpp:31-57,
 * 141-169): returns 0 = local, 1 = skip (a rank-bit control fails),
 * 2 = exchange with *peer; *ownLo = this rank owns the low half of each pair;
 * *lowMask = controls below the local qubit count. Returns -1 on invalid
 * input. */
int qgpuPlanGate(int flatQubits, int rankLog2, int rank, int target,
                 unsigned long long ctrlMask, int* peer, int* ownLo,
                 unsigned long long* lowMask);
/* Exchange schedule: number of sub-chunks and their size for a local length
 * and requested chunk (the PerAmplitude strategy with block = chunk,
 * distributed.cpp:215-231). */
int qgpuPlanChunks(unsigned long long localLen, unsigned long long chunkAmps,
                   unsigned long long* chunkLen);

/* Per-pass JIT of the fused tile pass: each distinct pass shape (op kinds,
 * qubit positions, control masks; not the angles) is compiled once with
 * NVRTC into straight-line code on background threads, and passes of that
 * shape use it from then on (results are identical to the interpreter).
 * mode 0 = off, 1 = background compiles (default; env QGPU_JIT=off|sync),
 * 2 = compile before the first launch of a shape. qgpuJitWait blocks until
 * every queued compile has finished; qgpuJitStats reports compiled kernels,
 * failures and pending compiles. */
void qgpuSetJit(int mode);
int qgpuGetJit(void);
void qgpuJitWait(void);
/* Stop the compile threads: queued shapes are dropped (they stay
 * interpreted), in-flight compiles finish, the JIT is off for the rest of
 * the process. Call before exit when compiles may be pending (the library
 * also does it from an atexit handler; the Python wrapper from its own). */
void qgpuJitShutdown(void);
void qgpuJitStats(unsigned long long* kernels, unsigned long long* failed, unsigned long long* pending);
/* Lane <-> register exchange ops the tile passes of this process have
 * carried so far (a run of pair ops on a lane qubit done in registers
 * between two exchanges instead of as warp-shuffle ops; QGPU_XCHG=0 turns
 * them off). A tuning / test counter. */
unsigned long long qgpuLaneExchanges(void);
/* Host-only (no GPU): compile a sample pass program for sm_100a with NVRTC.
 * Returns the cubin size, or -1 (message in log); *seconds = compile time. */
int qgpuJitSelfTest(char* log, int len, double* seconds);

/* Memory plan. The reference's node model, restated:
 * modeled peak bytes per rank of an n-qubit vector on 2^rankLog2 ranks for
 * strategy 0 = FullClone (2x), 1 = HalfExchange (1.5x), 2 = PerAmplitude
 * (1x + blockAmps), double or single precision
 * (qsim::modeled_bytes_per_rank, distributed.cpp:436-446; returns 0, or -1
 * on invalid input / 64-bit overflow), and the largest n that fits
 * nodeBytes - overheadBytes (qsim::max_qubits, distributed.cpp:448-468). */
int qgpuModeledBytesPerRank(int numQubits, int rankLog2, int strategy, int singlePrecision,
                            unsigned long long blockAmps, unsigned long long* bytes);
int qgpuMaxQubits(unsigned long long nodeBytes, unsigned long long overheadBytes, int strategy,
                  int singlePrecision, int rankLog2);
/* This runtime's device footprint per rank: the partition (16 B, or 8 B single, x
 * 2^(flat - k)), two exchange sub-chunk buffers of chunkAmps amplitudes once
 * k > 0, and the reduction scratch; and the largest register (qubits, or N
 * of an N-qubit density matrix) whose footprint fits deviceBytes.
 * createQureg preflights against free HBM with the same numbers. */
unsigned long long qgpuDeviceBytesPerRank(int flatQubits, int rankLog2, unsigned long long chunkAmps,
                                          int singlePrecision);
int qgpuDeviceMaxQubits(unsigned long long deviceBytes, int rankLog2, unsigned long long chunkAmps,
                        int density, int singlePrecision);

#ifdef __cplusplus
}
#endif

#endif /* QGPU_EXT_H */
