// runtime.h — host runtime of libqgpu: environment (device, streams,
// transport, RNG), registers (HBM shards), the op queue that fuses gates into
// HBM passes, the distributed exchange engine and the reductions.
#pragma once

#include "QuEST.h"
#include "qgpu.h"
#include "qgpu_device.h"
#include "swap_plan.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <set>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <vector>

namespace qgpu {

// Exceptions stay inside the library; api.cpp converts them to the error
// handler + codes (the reference's exception classes, types.hpp:31-55).
struct DomainError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ResourceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CommError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

void cuda_check(cudaError_t e, const char* what);
// cudaMemcpyAsync that adds host<->device bytes to the transfer counters
// (qgpuTransferBytes: the bench's e2e h2d / d2h bytes per step)
cudaError_t memcpy_counted(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s);

// ------------------------------------------------------------- transport

class NcclComm;  // transport.cpp
class PeerGroup; // peer.cpp

// Single: one GPU. Loopback: 2^k virtual ranks on one GPU. Nccl: one process
// per GPU over NCCL send/recv. Peer: one process per GPU of one node, every
// partition mapped into every rank (CUDA IPC over NVLink; peer.h).
enum class Mode { Single, Loopback, Nccl, Peer };

struct Env {
    int device = 0;
    cudaStream_t stream = nullptr;      // all compute
    cudaStream_t comm_stream = nullptr; // NCCL sends/recvs
    Mode mode = Mode::Single;
    int rank = 0;        // this process's rank (Nccl) or 0
    int num_ranks = 1;   // total ranks (virtual ranks in Loopback)
    int rank_log2 = 0;
    uint64_t rng = 0;    // SplitMix64 state for measure()
    int fusion_mode = 0; // 0 fused, 1 one pass per op, 2 simple per-op kernels
    int max_ops = kMaxPassOps;      // register-only passes (small states)
    int tile_max_ops = kMaxTileOps; // tile passes (qgpuSetFusion's maxOps sets both)
    int reg_qubits = 4;
    // tile-pass shape limits (scheduler tuning; QGPU_TILE_TARGETS /
    // QGPU_TILE_PHASES override them at Env creation). A phase transition
    // (a shared-memory round trip of the whole tile plus a barrier) costs
    // about three interpreted ops or five JIT ops, and a fresh pass is free
    // while the pass stays HBM-bound: measured on the 30-qubit layered
    // circuit, at most two phases per pass is fastest for the interpreter and
    // three under the JIT (profiles/r1_scheduler_knobs.md; max_phases()).
    int tile_targets = kTileHigh; // distinct pair targets above qubit 4 per pass
    int tile_phases = 0;          // register phases per pass (0: by JIT mode)
    uint64_t chunk_amps = uint64_t{1} << 24;
    // global<->local qubit swaps instead of per-gate exchanges (swap_plan.h);
    // qgpuSetQubitSwaps turns them off (the reference's exchange per gate)
    bool qubit_swaps = true;
    // op order inside the tile passes (qgpuSetOrdering / QGPU_ORDER):
    // 1 (default) schedules commuting ops out of circuit order into fewer
    // passes (amplitudes within 1e-12 of the reference, not bit-identical);
    // 0 keeps circuit order (bit-identical to the reference)
    int order = 1;
    int window = 512; // ops the reorder scheduler looks ahead (QGPU_WINDOW)
    // shuffle lane ops per reordered pass (QGPU_LANE_CAP; 0: no cap): capped,
    // they spread over passes where the shuffle unit idles instead of making
    // two or three passes shuffle-bound (30q bench: 162.9 vs 165.3 ms/step
    // uncapped, cap 12: 165.3; profiles/r2/r2y)
    int lane_cap = 8;
    int normalize = 1;   // unit-coefficient gate normalization in tolerance mode (QGPU_NORMALIZE)
    int merge = 1;       // same-qubit gate merging in the reorder window (QGPU_MERGE)
    // lane <-> register exchanges around runs of lane-qubit pair ops (QGPU_XCHG:
    // 1 with room reserved in reordered passes, 2 where a pass has room; off:
    // measured slower on the bench circuit, the per-element selects of an
    // exchange cost more ALU issue than the shuffles they save)
    int exchanges = 0;
    // swizzled middle phases (QGPU_SWIZZLE=<n>): a reordered pass with at
    // least n pair ops on qubits 0-2 gets a middle phase holding them as
    // register qubits (tile_body.inc: TilePhase.swz); 0 = off. 30q bench:
    // 154.1 ms per step at n = 6, 155.7 at 3, 164.8 off (profiles/r2/r2sw)
    int swizzle = 6;
    std::unique_ptr<NcclComm> nccl;
    std::unique_ptr<PeerGroup> peer;
    bool multi_process() const { return mode == Mode::Nccl || mode == Mode::Peer; }
    // smallest contiguous block a global<->local swap should trade (swap
    // victims sit at positions >= its log2): the sub-chunk of the send /
    // receive transports; the peer kernel moves blocks of 2^5 amplitudes
    // (coalesced warps), which keeps victims off the lane qubits 0-4 (a
    // global qubit landing there would make its gates shuffle ops) while
    // the light-cone drain can evict the low qubits whose work is done
    uint64_t swap_granule() const { return mode == Mode::Peer ? 32 : chunk_amps; }
    std::set<struct QuregImpl*> quregs;

    // Launch profiling (qgpuProfileStart/Stop): an event pair around every
    // launch of the hot kernels, on the stream they run on.
    bool profile = false;
    struct ProfRec {
        cudaEvent_t start, stop;
        int kind;
        int info; // PK_PASS: ops | phases << 16
    };
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> event_pool;
    cudaEvent_t take_event();
    // cudaStreamSynchronize that, on NCCL ranks, polls ncclCommGetAsyncError
    // and gives up after QGPU_NCCL_TIMEOUT_S (a partner that died or threw
    // would otherwise leave this rank blocked inside NCCL forever)
    void wait_stream(cudaStream_t s);

    ~Env();
};

enum ProfKind { PK_PASS = 0, PK_SIMPLE = 1, PK_EXCHANGE = 2, PK_DEPOL = 3, PK_REDUCE = 4, PK_SWAP = 5 };

// Brackets the enclosed launches with an event pair when profiling is on.
class ProfScope {
  public:
    ProfScope(Env* env, int kind, int info = 0);
    ~ProfScope();

  private:
    Env* env_;
    int kind_;
    int info_;
    cudaEvent_t start_ = nullptr;
};

// --------------------------------------------------------------- registers

enum FlatKind : uint8_t { FK_GATE = 0, FK_DEPHASE = 1, FK_DEPOL = 2, FK_COLLAPSE = 3 };

// An operation on the flat 2^flat vector (the reference's FlatGateOp,
// distributed.hpp:78-85, extended with the channels and collapse).
// lane <-> register exchange ops emitted by tile passes (qgpuLaneExchanges)
extern std::atomic<unsigned long long> g_lane_exchanges;

struct FlatOp {
    uint8_t kind = FK_GATE;
    uint8_t cls = CLS_GENERIC;
    uint8_t flags = 0;
    uint8_t outcome = 0;
    int q0 = 0, q1 = -1;
    uint64_t cmask = 0;
    double m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int32_t id = -1; // caller's op index (qgpuPlanPasses dry runs)
    // unit coefficients of a normalized real / Rx-class gate (tolerance mode,
    // runtime.cpp normalize_op): 2 bits per coefficient, tile header bits 40-47
    uint8_t unit = 0;
};

uint8_t classify(const double* m, uint8_t* diag_flags);

struct Shard {
    int rank = 0;
    void* amps = nullptr; // double2[local_len], or float2[local_len] for single precision
    uint64_t messages = 0, bytes = 0; // CommStats per rank
};

struct QuregImpl {
    Env* env = nullptr;
    int N = 0;          // qubits represented
    int flat = 0;       // N (SV) or 2N (DM)
    bool density = false;
    bool single = false; // Precision::Single: float2 amplitudes, float arithmetic
    int local_qubits = 0;
    uint64_t local_len = 0;
    std::vector<Shard> shards; // 1, or 2^k virtual ranks (Loopback)
    std::vector<void*> peer_amps; // Peer: every rank's partition mapped here ([rank] = shards[0])
    void* recv[2] = {nullptr, nullptr};
    uint64_t recv_len = 0;
    double2* partials = nullptr; // reduction scratch
    double2* results = nullptr;  // one (hi, lo) per shard
    uint64_t passes = 0;

    size_t amp_bytes() const { return single ? sizeof(float2) : sizeof(double2); }
    // qubits held by fixed lane bits in every tile phase: 0-2, and 3 in single
    // precision (runtime.cpp: launch_tile's shared-memory bank argument)
    int lane_fixed() const { return pin_lane3() ? kFixedLaneBits + 1 : kFixedLaneBits; }
    bool pin_lane3() const;
    // element `i` of a shard (or exchange buffer) as a byte address
    char* at(void* base, uint64_t i) const { return static_cast<char*>(base) + i * amp_bytes(); }

    // the open pass
    std::vector<FlatOp> pending;
    std::vector<int> regs; // register qubits (small-state register pass)
    struct PhaseState {
        std::vector<int> regs; // register qubits of the phase
        int op_begin = 0;
        bool mid = false; // swizzled middle phase: qubits 0-2 are register qubits
    };
    std::vector<int> tile_high;      // tile pass: high qubits in the tile
    std::vector<PhaseState> phases;  // tile pass: phases

    // Reorder window (Env::order == 1, tile passes): physical ops awaiting
    // pass formation. A pass is cut from the window by commutation, not by
    // position (window_pass); pending / phases then hold that pass only.
    std::vector<FlatOp> win;
    // Scalar factored out of the window's normalized gates (normalize_op),
    // folded into one op of a later pass (fold_scale); 1 whenever the window
    // is empty after a drain.
    double gscale_re = 1.0, gscale_im = 0.0;
    bool normalize_op(FlatOp& op);
    bool merge_into_window(const FlatOp& op);
    std::unordered_map<int, std::vector<int>> merged_ids; // dry runs: ids merged into an op
    bool fold_scale();
    bool reorder_on() const;
    void window_pass();  // form and launch one pass from the window
    void window_drain(); // ... until the window is empty

    // Dry run (qgpuPlanPasses): passes are recorded here instead of launched
    struct PlannedPass {
        std::vector<int> ids;         // FlatOp::id in execution order
        std::vector<int> phase_begin; // index into ids where each phase starts
    };
    std::vector<PlannedPass>* plan_sink = nullptr;
    std::vector<std::pair<int, int>>* swap_sink = nullptr; // dry runs: (global, local) swaps

    // logical -> physical qubit map (global<->local swaps, swap_plan.h)
    SwapPlanner sp;

    ~QuregImpl();

    // queue an op on LOGICAL qubits: maps it through the swap planner (and
    // swaps a global target in first), then enqueue_phys
    void enqueue(const FlatOp& op);
    void enqueue_phys(const FlatOp& op);
    std::vector<FlatOp> lq;       // logical ops awaiting swap planning
    void drain(size_t count);     // plan + enqueue_phys the first `count` of lq
    void drain_lightcone(size_t count); // (reordering mode: any runnable ops first)
    void flush_pass();            // launch the open pass
    bool swaps_on() const { return env->qubit_swaps && env->rank_log2 > 0; }
    // move every logical qubit back to its own position (before amplitudes
    // are read or written by index)
    void restore_identity();
    void flush();
    void discard_all() { // queued ops are dead (the state is overwritten)
        lq.clear();
        win.clear();
        gscale_re = 1.0;
        gscale_im = 0.0;
        deferred.clear();
        ++version;
        discard();
    }

    // ---- measurement support (state vectors)
    // Every mutation bumps `version`; the single-qubit marginals of the
    // current state are computed in one read (launch_marginals) and serve
    // every calcProbOfOutcome / measure until the next mutation.
    uint64_t version = 0;
    uint64_t marg_version = ~uint64_t{0};
    std::vector<double2> marg;       // [0] total, [1 + L] sum over logical qubit L == 1 (double-double)
    void* marg_scratch = nullptr;    // launch_marginals scratch (lazy)
    double2* marg_dev = nullptr;     // per-shard / per-rank marginal vectors
    bool marginals_usable() const;
    void compute_marginals();
    // Collapses of a state vector wait here while only reductions follow:
    // a probability (or the total) is then a reduction over the amplitudes
    // the pending collapses keep (a fraction of the state) times their
    // scale^2, and the collapses themselves fuse into the next pass. Any
    // other op, read or write enqueues them first, in order.
    std::vector<FlatOp> deferred;    // logical FK_COLLAPSE ops
    void defer_collapse(const FlatOp& op);
    void materialize();
    // sum |a|^2 over the physical selection (mask, val), all shards, rank order
    double reduce_sel_phys(uint64_t mask, uint64_t val);
    void discard() {
        pending.clear();
        regs.clear();
        tile_high.clear();
        phases.clear();
    }

    // reductions (flush first; synchronous)
    double reduce_norm(int t, int outcome); // sum |a|^2 (t < 0: all)
    double reduce_diag(int t, int outcome, int comp = 0); // sum Re (comp 0) / Im (1) rho_jj
    Complex trace();

    void get_flat(uint64_t start, uint64_t num, double2* out);
    void set_flat(uint64_t start, uint64_t num, const double2* in);
    void fill_zero();

  private:
    int pass_H() const;
    bool use_tile() const;
    bool place_tile(const FlatOp& op, bool pair);
    bool place_tile_depol(const FlatOp& op);
    int max_phases() const;
    void launch_tile();
    void run_simple(const FlatOp& op);
    void launch_fused();
    void run_exchange_gate(const FlatOp& op);
    void run_depol(const FlatOp& op);
    // trade physical global position g with local v; flush = false: only the
    // open pass runs first (the caller ran the window's ops on g and v)
    void run_swap(int g, int v, bool flush = true);
    void local_swap(int a, int b);
    void ensure_recv(uint64_t len);
    uint64_t goff(const Shard& s) const { return static_cast<uint64_t>(s.rank) * local_len; }
    double combine_results(int n); // rank-ordered double-double sum
    // amplitude bytes in the register's own precision (get_flat / set_flat
    // convert at the host boundary)
    void get_raw(uint64_t start, uint64_t num, void* out);
    void set_raw(uint64_t start, uint64_t num, const void* in);
};

QuregImpl* create_register(Env* env, int N, bool density, bool single = false);

bool pass_stats_enabled();
void record_pass_stats(const TileParams& P);

// Pure planner (qgpu.h: qgpuPlanGate).
// memory_plan.cpp: the reference's node model (distributed.cpp:423-468) and
// this runtime's per-rank device footprint
uint64_t modeled_bytes_per_rank(int n, int k, int strategy, bool single, uint64_t block);
int max_qubits(uint64_t node_bytes, uint64_t overhead, int strategy, bool single, int k);
uint64_t device_bytes_per_rank(int flat, int k, uint64_t chunk_amps, bool single = false);
int device_max_qubits(uint64_t device_bytes, int k, uint64_t chunk_amps, bool density,
                      bool single = false);

int plan_gate(int flat, int rank_log2, int rank, int target, uint64_t cmask, int* peer,
              int* own_lo, uint64_t* low_mask);

} // namespace qgpu
