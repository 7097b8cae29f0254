// runtime.cpp — registers in HBM, the fused-pass scheduler, the distributed
// exchange engine and the compensated reductions.
//
// Reference mapping (paths under /root/reference/proj):
//   QuregImpl / create_register     Register ctor + init, register.cpp:101-130
//   enqueue/flush/launch_fused      run_circuit's op-by-op dispatch,
//                                   circuit.cpp:239-247, fused into HBM passes
//   run_simple                      apply_gate_span, kernels.cpp:43-59
//   plan_gate                       partition / needs_communication /
//                                   pair_rank, distributed.cpp:31-57, 141-169
//   run_exchange_gate               rank_apply_op exchange + combine,
//                                   distributed.cpp:167-231 (PerAmplitude
//                                   strategy with block = sub-chunk)
//   run_depol                       depolarising_pass, density.cpp:62-81
//                                   (+ its distribution, absent upstream)
//   reduce_norm / reduce_diag       norm_squared register.cpp:62-75, trace
//                                   density.cpp:147-154 (compensated)
#include "runtime.h"

#include "peer.h"
#include "qgpu_kernels.h"
#include "transport.h"

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <cstring>

namespace qgpu {

std::atomic<unsigned long long> g_lane_exchanges{0};

cudaError_t memcpy_counted(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    if (kind == cudaMemcpyHostToDevice) count_transfer(bytes, 0);
    if (kind == cudaMemcpyDeviceToHost) count_transfer(0, bytes);
    return cudaMemcpyAsync(dst, src, bytes, kind, s);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

Env::~Env() {
    for (QuregImpl* q : std::vector<QuregImpl*>(quregs.begin(), quregs.end())) delete q;
    nccl.reset();
    peer.reset();
    for (auto& r : prof) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (comm_stream) cudaStreamDestroy(comm_stream);
}

void Env::wait_stream(cudaStream_t s) {
    if (!nccl) {
        cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        return;
    }
    static const double timeout_s = [] {
        const char* v = std::getenv("QGPU_NCCL_TIMEOUT_S");
        return v ? std::max(1.0, std::atof(v)) : 600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) cuda_check(e, "cudaStreamQuery");
        nccl->check_async();
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
            nccl->abort();
            throw CommError("rank " + std::to_string(rank) + " timed out waiting for NCCL (QGPU_NCCL_TIMEOUT_S)");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

cudaEvent_t Env::take_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

ProfScope::ProfScope(Env* env, int kind, int info) : env_(env), kind_(kind), info_(info) {
    if (!env_->profile) return;
    start_ = env_->take_event();
    cuda_check(cudaEventRecord(start_, env_->stream), "cudaEventRecord");
}

ProfScope::~ProfScope() {
    if (!start_) return;
    cudaEvent_t stop = env_->take_event();
    cudaEventRecord(stop, env_->stream);
    env_->prof.push_back({start_, stop, kind_, info_});
}

uint8_t classify(const double* m, uint8_t* diag_flags) {
    auto z = [&](int k) { return m[k] == 0.0; };
    *diag_flags = 0;
    if (z(2) && z(3) && z(4) && z(5)) {
        if (m[0] == 1.0 && z(1)) *diag_flags |= DF_A_ONE;
        if (m[6] == 1.0 && z(7)) *diag_flags |= DF_D_ONE;
        return CLS_DIAG;
    }
    if (z(0) && z(1) && m[2] == 1.0 && z(3) && m[4] == 1.0 && z(5) && z(6) && z(7))
        return CLS_SWAP;
    if (z(1) && z(3) && z(5) && z(7)) return CLS_REAL;
    if (z(1) && z(2) && z(4) && z(7)) return CLS_RX;
    return CLS_GENERIC;
}

int plan_gate(int flat, int rank_log2, int rank, int target, uint64_t cmask, int* peer,
              int* own_lo, uint64_t* low_mask) {
    if (flat < 1 || rank_log2 < 0 || rank_log2 > flat || target < 0 || target >= flat ||
        rank < 0 || rank >= (1 << rank_log2) || ((cmask >> target) & 1u) ||
        (flat < 64 && (cmask >> flat)))
        return -1;
    const int m = flat - rank_log2;
    const uint64_t local_len = uint64_t{1} << m;
    *low_mask = cmask & (local_len - 1);
    *peer = rank;
    *own_lo = 1;
    // distributed.cpp:141-145: rank-bit controls resolved from the rank id.
    const uint64_t rank_mask = m >= 64 ? 0 : (cmask >> m);
    if ((static_cast<uint64_t>(rank) & rank_mask) != rank_mask) return 1;
    if (target < m) return 0; // distributed.cpp:161-165
    const int rank_bit = target - m;
    *peer = rank ^ (1 << rank_bit);                  // distributed.cpp:50-57
    *own_lo = ((rank >> rank_bit) & 1) == 0 ? 1 : 0; // distributed.cpp:169
    return 2;
}

// ---------------------------------------------------------------- register

QuregImpl* create_register(Env* env, int N, bool density, bool single) {
    if (N < 1)
        throw DomainError("register needs at least 1 qubit, got " + std::to_string(N));
    const int flat = density ? 2 * N : N;
    // register.cpp:106-117: preflight the byte count.
    if (flat + 4 > 63)
        throw ResourceError("register of " + std::to_string(N) + " qubits requires 2^" +
                            std::to_string(flat + 4) + " bytes");
    if (env->rank_log2 > flat)
        throw DomainError("rank count 2^" + std::to_string(env->rank_log2) + " invalid for " +
                          std::to_string(flat) + " qubits (need 0 <= k <= n)");
    if (density && env->rank_log2 > N)
        throw DomainError("density matrix of " + std::to_string(N) +
                          " qubits cannot be split over 2^" + std::to_string(env->rank_log2) +
                          " ranks (need k <= N)");
    // preflight against free HBM (an infeasible size is a
    // resource error citing max_qubits)
    {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            const int nsh = env->mode == Mode::Loopback ? env->num_ranks : 1;
            const uint64_t per = device_bytes_per_rank(flat, env->rank_log2, env->chunk_amps, single);
            const unsigned __int128 need = static_cast<unsigned __int128>(per) * nsh;
            if (need > free_b) {
                const int mq = device_max_qubits(free_b / nsh, env->rank_log2, env->chunk_amps, density, single);
                throw ResourceError("register of " + std::to_string(N) + " qubits needs " +
                                    std::to_string(per) + " bytes per rank but " +
                                    std::to_string(free_b) + " bytes of device memory are free: " +
                                    "max_qubits = " + std::to_string(mq) + " at 2^" +
                                    std::to_string(env->rank_log2) + " ranks");
            }
        } else {
            cudaGetLastError();
        }
    }
    auto q = std::make_unique<QuregImpl>();
    q->env = env;
    q->N = N;
    q->flat = flat;
    q->density = density;
    q->single = single;
    q->local_qubits = flat - env->rank_log2;
    q->local_len = uint64_t{1} << q->local_qubits;
    const int nshards = env->mode == Mode::Loopback ? env->num_ranks : 1;
    const size_t bytes = q->local_len * q->amp_bytes();
    for (int s = 0; s < nshards; ++s) {
        Shard sh;
        sh.rank = env->mode == Mode::Loopback ? s : env->rank;
        if (cudaMalloc(&sh.amps, bytes) != cudaSuccess) {
            cudaGetLastError();
            throw ResourceError("failed to allocate " + std::to_string(bytes) +
                                " bytes of amplitude storage");
        }
        q->shards.push_back(sh);
    }
    if (env->mode == Mode::Peer) {
        try {
            q->peer_amps = env->peer->open_all(q->shards[0].amps);
        } catch (...) {
            cudaFree(q->shards[0].amps);
            q->shards.clear();
            throw;
        }
    }
    const int nresults = std::max(nshards, env->num_ranks) + 1;
    if (cudaMalloc(&q->partials, kReduceBlocks * sizeof(double2)) != cudaSuccess ||
        cudaMalloc(&q->results, nresults * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        throw ResourceError("failed to allocate reduction scratch");
    }
    q->sp.reset(flat, q->local_qubits, env->swap_granule());
    q->fill_zero();
    if (q->shards[0].rank == 0) {
        const double2 one = make_double2(1.0, 0.0);
        const float2 one_f = make_float2(1.0f, 0.0f);
        cuda_check(memcpy_counted(q->shards[0].amps, single ? static_cast<const void*>(&one_f) : &one,
                                   q->amp_bytes(), cudaMemcpyHostToDevice, env->stream),
                   "init zero state");
        cuda_check(cudaStreamSynchronize(env->stream), "init zero state");
    }
    env->quregs.insert(q.get());
    return q.release();
}

QuregImpl::~QuregImpl() {
    if (env) {
        cudaStreamSynchronize(env->stream);
        env->quregs.erase(this);
        if (env->peer && !peer_amps.empty()) env->peer->close_all(peer_amps); // collective
    }
    for (auto& s : shards) cudaFree(s.amps);
    cudaFree(recv[0]);
    cudaFree(recv[1]);
    cudaFree(partials);
    cudaFree(results);
    cudaFree(marg_scratch);
    cudaFree(marg_dev);
}

void QuregImpl::fill_zero() {
    discard_all();
    for (auto& s : shards)
        cuda_check(cudaMemsetAsync(s.amps, 0, local_len * amp_bytes(), env->stream),
                   "cudaMemsetAsync");
    sp.reset(flat, local_qubits, env->swap_granule()); // the whole state is rewritten
}

void QuregImpl::ensure_recv(uint64_t len) {
    if (recv_len >= len) return;
    cuda_check(cudaStreamSynchronize(env->stream), "sync");
    cudaFree(recv[0]);
    cudaFree(recv[1]);
    recv[0] = recv[1] = nullptr;
    recv_len = 0;
    if (cudaMalloc(&recv[0], len * amp_bytes()) != cudaSuccess ||
        cudaMalloc(&recv[1], len * amp_bytes()) != cudaSuccess) {
        cudaGetLastError();
        throw ResourceError("failed to allocate " + std::to_string(2 * len * amp_bytes()) +
                            " bytes of exchange buffers");
    }
    recv_len = len;
}

int QuregImpl::pass_H() const {
    const int h = std::min(std::min(env->reg_qubits, 3), local_qubits - kLaneQubits);
    return h < 1 ? 0 : h;
}

bool QuregImpl::use_tile() const { return local_qubits >= kTileQubits; }

// -------------------------------------------------------------- scheduling
//
// Ops are queued in order and cut into passes; no op is ever reordered, so
// every amplitude sees exactly the reference's sequence of operations.
// Tile mode (>= 12 local qubits): a pass may touch the 5 lane qubits plus
// kTileHigh other qubits; inside it, a phase may pair on the lanes plus
// kPhaseRegBits register qubits. Diagonal gates, dephasing and collapse act
// elementwise and fit anywhere.

// Phases per pass: QGPU_TILE_PHASES / Env::tile_phases if set, else 3 when
// the per-pass JIT is on and 2 for the interpreter (profiles/: a transition
// costs ~3 interpreted ops but only ~5 straight-line ones).
int QuregImpl::max_phases() const {
    if (env->tile_phases > 0) return env->tile_phases;
    return jit_mode() != 0 ? 3 : 2;
}

// single precision keeps tile bit 3 on lane bit 3 (QGPU_SP_PIN3=0 turns it
// off: an A/B knob)
bool QuregImpl::pin_lane3() const {
    static const bool on = [] {
        const char* e = std::getenv("QGPU_SP_PIN3");
        return !(e && e[0] == '0');
    }();
    return single && on;
}

bool QuregImpl::place_tile(const FlatOp& op, bool pair) {
    if (phases.empty()) phases.push_back(PhaseState{});
    if (pair && op.q0 >= lane_fixed()) {
        const int q = op.q0;
        PhaseState& ph = phases.back();
        const bool in_phase = std::find(ph.regs.begin(), ph.regs.end(), q) != ph.regs.end();
        if (q < kLaneQubits) {
            // qubits 3, 4: a register qubit if the phase has room, else a
            // lane qubit of this phase (a shuffle op; a new phase costs more)
            if (!in_phase && static_cast<int>(ph.regs.size()) < kPhaseRegBits) ph.regs.push_back(q);
        } else {
            const bool in_tile = std::find(tile_high.begin(), tile_high.end(), q) != tile_high.end();
            if (!in_tile && static_cast<int>(tile_high.size()) >= env->tile_targets) return false;
            // a phase holds kPhaseRegBits register qubits
            if (!in_phase && static_cast<int>(ph.regs.size()) >= kPhaseRegBits) {
                if (static_cast<int>(phases.size()) >= max_phases()) return false;
                PhaseState next;
                next.op_begin = static_cast<int>(pending.size());
                phases.push_back(next);
            }
            if (!in_phase) phases.back().regs.push_back(q);
            if (!in_tile) tile_high.push_back(q);
        }
    }
    pending.push_back(op);
    return true;
}

// A depolarising channel needs both its qubits as register qubits of one
// phase (its 4-groups span both bits).
bool QuregImpl::place_tile_depol(const FlatOp& op) {
    if (phases.empty()) phases.push_back(PhaseState{});
    auto has = [](const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); };
    int new_high = 0;
    for (int q : {op.q0, op.q1})
        if (q >= kLaneQubits && !has(tile_high, q)) ++new_high;
    if (static_cast<int>(tile_high.size()) + new_high > env->tile_targets) return false;
    PhaseState* ph = &phases.back();
    // register qubits it needs: both, or only t+N when t is a fixed lane bit
    std::vector<int> regq;
    if (op.q0 >= lane_fixed()) regq.push_back(op.q0);
    regq.push_back(op.q1);
    int need = 0;
    for (int q : regq)
        if (!has(ph->regs, q)) ++need;
    if (static_cast<int>(ph->regs.size()) + need > kPhaseRegBits) {
        if (static_cast<int>(phases.size()) >= max_phases()) return false;
        PhaseState next;
        next.op_begin = static_cast<int>(pending.size());
        phases.push_back(next);
        ph = &phases.back();
    }
    for (int q : regq) {
        if (!has(ph->regs, q)) ph->regs.push_back(q);
        if (q >= kLaneQubits && !has(tile_high, q)) tile_high.push_back(q);
    }
    pending.push_back(op);
    return true;
}

// ------------------------------------------------------- reorder scheduler
//
// Env::order == 1 (the default). Physical ops wait in a window of up to
// Env::window; a pass takes a subset of them that is closed under "must
// precede" and fits one tile pass, in an order consistent with it. Op j
// must follow an earlier op i when they share a qubit on which at least one
// of them acts non-diagonally (a pair target, a depolarising qubit);
// controls, diagonal targets, dephasing and collapse act diagonally on
// their qubits, and ops that only meet on such qubits commute. Commuting ops
// are exchangeable in exact arithmetic, so the state equals the
// circuit-order one up to rounding (tests/test_gpu_reorder.py: within 1e-12
// of the reference's amplitudes at 30 qubits) — not bit for bit: Env::order
// = 0 keeps circuit order and bit-identity.
//
// Per pass: the tile's high qubits are picked greedily, each time the qubit
// whose addition lets the most window ops into the pass (a closure computed
// in one ordered scan with blocked-qubit masks); then the selected ops are
// list-scheduled into phases: every ready op that fits the phase's register
// qubits runs, and when none does the phase takes the register qubit that
// unblocks the most ready ops; a phase ends when its registers are full and
// nothing else fits. Ops the phases could not take stay in the window.
namespace {
// How an op acts on each qubit, for commutation: diagonally (controls,
// diagonal targets, dephasing, collapse), as an X-type 2x2 ([[a, b], [b,
// a]]: X / CNOT targets, Rx — these commute with each other), or otherwise
// non-diagonally. Two ops commute when every qubit they share is diagonal
// in both or X-type in both.
struct OpQubits {
    uint64_t nd = 0;   // qubits the op acts on non-diagonally, not X-type
    uint64_t nx = 0;   // qubits it acts on as an X-type 2x2
    uint64_t dg = 0;   // qubits it acts on diagonally (controls, phases)
    uint64_t need = 0; // qubits that must be in the tile
};
bool x_type(const FlatOp& op) {
    return op.kind == FK_GATE && op.cls != CLS_DIAG && op.m[0] == op.m[6] && op.m[1] == op.m[7] &&
           op.m[2] == op.m[4] && op.m[3] == op.m[5];
}
OpQubits op_qubits(const FlatOp& op) {
    auto bit = [](int q) { return q >= 0 ? uint64_t{1} << q : uint64_t{0}; };
    OpQubits r;
    if (op.kind == FK_GATE) {
        r.dg = op.cmask;
        if (op.cls == CLS_DIAG) {
            r.dg |= bit(op.q0);
        } else {
            (x_type(op) ? r.nx : r.nd) = bit(op.q0);
            r.need = bit(op.q0);
        }
    } else if (op.kind == FK_DEPOL) {
        r.nd = bit(op.q0) | bit(op.q1);
        r.need = r.nd;
    } else { // dephasing, collapse: elementwise
        r.dg = bit(op.q0) | bit(op.q1);
    }
    return r;
}
// what the ops skipped so far act on (an op may not pass any of them that it
// does not commute with)
struct Blockers {
    uint64_t nd = 0, nx = 0, dg = 0;
    void add(const OpQubits& o) {
        nd |= o.nd;
        nx |= o.nx;
        dg |= o.dg;
    }
};
inline bool blocked_by(const OpQubits& a, const Blockers& b) {
    return (a.nd & (b.nd | b.nx | b.dg)) != 0 || (a.nx & (b.nd | b.dg)) != 0 || (a.dg & (b.nd | b.nx)) != 0;
}
} // namespace

// Unit-coefficient normalization (tolerance mode): an uncontrolled real or
// Rx-class gate is its largest-magnitude coefficient v times a matrix whose
// entries include exact +-1 (H -> [[1, 1], [1, -1]] and 1/sqrt 2; Ry(t) ->
// [[1, -tan], [tan, 1]] and cos, or [[cot, -1], [1, cot]] and -sin; Rx
// alike with i), and an uncontrolled diagonal is a times diag(1, d / a) (Rz
// -> diag(1, e^{i theta}) and e^{-i theta / 2}). The kernels skip the
// multiplications by +-1 (tile header unit bits) and the identity half of a
// diagonal: roughly half the FP64 work of the layered circuit. The scalars
// commute with every linear op, so they are multiplied together and applied
// once, folded into one op of some pass (fold_scale) — before the window
// drains empty, i.e. before anything reads the state.
bool QuregImpl::normalize_op(FlatOp& op) {
    if (op.kind != FK_GATE || op.cmask != 0) return false;
    double* m = op.m;
    double vr, vi;
    if (op.cls == CLS_DIAG) {
        const double ar = m[0], ai = m[1], den = ar * ar + ai * ai;
        if (!(den > 0.0)) return false;
        const double dr = (m[6] * ar + m[7] * ai) / den, di = (m[7] * ar - m[6] * ai) / den;
        if (env->normalize == 1 && op.q0 < lane_fixed() && std::fabs(dr * dr + di * di - 1.0) < 1e-14 &&
            dr > -0.999) {
            // On a fixed lane qubit every lane multiplies by its side's factor,
            // so the identity side of diag(1, r) still costs a complex product.
            // Symmetric form instead: diag(1, r) = s diag(1 - it, 1 + it) with
            // t = tan(arg(r) / 2), s = 1 / (1 - it): unit real parts, two FMAs
            // per amplitude on both sides (unit bit 0: h_diag_lane_fast).
            const double t = di / (1.0 + dr), q = 1.0 / (1.0 + t * t);
            const double sr = q, si = t * q; // 1 / (1 - it) = (1 + it) / (1 + t^2)
            vr = ar * sr - ai * si;
            vi = ar * si + ai * sr;
            m[0] = 1.0;
            m[1] = -t;
            m[6] = 1.0;
            m[7] = t;
            op.flags = 0;
            op.unit = 1; // real parts exactly 1
        } else {
            if (op.flags & DF_A_ONE) return false;
            vr = ar;
            vi = ai;
            m[0] = 1.0;
            m[1] = 0.0;
            m[6] = dr;
            m[7] = di;
            op.flags = DF_A_ONE | ((dr == 1.0 && di == 0.0) ? DF_D_ONE : 0);
        }
    } else if (op.cls == CLS_REAL || op.cls == CLS_RX) {
        static const int kReal[4] = {0, 2, 4, 6}, kRx[4] = {0, 3, 5, 6};
        const int* idx = op.cls == CLS_REAL ? kReal : kRx;
        double v = m[idx[0]];
        for (int k = 1; k < 4; ++k)
            if (std::fabs(m[idx[k]]) > std::fabs(v)) v = m[idx[k]];
        if (!(std::fabs(v) > 0.0) || !std::isfinite(v)) return false;
        uint8_t unit = 0;
        for (int k = 0; k < 4; ++k) {
            m[idx[k]] /= v;
            if (m[idx[k]] == 1.0) unit |= static_cast<uint8_t>(1u << (2 * k));
            if (m[idx[k]] == -1.0) unit |= static_cast<uint8_t>(2u << (2 * k));
        }
        op.unit = unit;
        vr = v;
        vi = 0.0;
    } else {
        return false;
    }
    const double r = gscale_re * vr - gscale_im * vi, i = gscale_re * vi + gscale_im * vr;
    gscale_re = r;
    gscale_im = i;
    return true;
}

// Applies the pending scalar to one uncontrolled gate of the open pass,
// the cheapest available: a generic 2x2 (free), a diagonal (its identity
// half comes back), a real / Rx-class gate (loses its unit entries; becomes
// generic if the scalar is complex). Returns false if the pass has none.
bool QuregImpl::fold_scale() {
    if (gscale_re == 1.0 && gscale_im == 0.0) return true;
    int best = -1, best_cost = 1 << 30;
    for (size_t k = 0; k < pending.size(); ++k) {
        const FlatOp& op = pending[k];
        if (op.kind != FK_GATE || op.cmask != 0) continue;
        int cost;
        if (op.cls == CLS_GENERIC) cost = 0;
        else if (op.cls == CLS_DIAG) cost = 2;
        else if (op.cls == CLS_REAL || op.cls == CLS_RX) cost = gscale_im == 0.0 ? 2 : 6;
        else continue; // swaps stay pure moves
        if (cost < best_cost) {
            best_cost = cost;
            best = static_cast<int>(k);
        }
    }
    if (best < 0) return false;
    FlatOp& op = pending[best];
    const double sr = gscale_re, si = gscale_im;
    op.unit = 0; // the unit entries take the scalar (they were exact)
    if ((op.cls == CLS_REAL || op.cls == CLS_RX) && si != 0.0) op.cls = CLS_GENERIC;
    for (int k = 0; k < 8; k += 2) {
        const double a = op.m[k], b = op.m[k + 1];
        op.m[k] = a * sr - b * si;
        op.m[k + 1] = a * si + b * sr;
    }
    if (op.cls == CLS_DIAG) {
        op.flags = 0;
        if (op.m[0] == 1.0 && op.m[1] == 0.0) op.flags |= DF_A_ONE;
        if (op.m[6] == 1.0 && op.m[7] == 0.0) op.flags |= DF_D_ONE;
    }
    gscale_re = 1.0;
    gscale_im = 0.0;
    return true;
}

bool QuregImpl::reorder_on() const {
    return env->order == 1 && use_tile() && env->fusion_mode == 0;
}

// Same-qubit merging (tolerance mode): an uncontrolled 2x2 gate X on qubit q
// is multiplied into the latest window op Y on q that is itself an
// uncontrolled 2x2 on q, provided X commutes with every op in between that
// touches q (op_qubits' rule: diagonal with diagonal, X-type with X-type) and
// the product stays a cheap class (diagonal, real or Rx-class: Rz Rz, Rx Rx
// across CNOT targets, Ry Ry, ...; a complex 2x2 costs more than the two
// rotations). Y then applies X Y at Y's place — X moved across ops it
// commutes with. Dry runs record X's id after Y's (merged_ids).
bool QuregImpl::merge_into_window(const FlatOp& x) {
    if (x.kind != FK_GATE || x.cmask != 0 || win.empty()) return false;
    const OpQubits xo = op_qubits(x);
    const uint64_t qb = uint64_t{1} << x.q0;
    for (size_t k = win.size(); k-- > 0;) {
        FlatOp& y = win[k];
        const OpQubits yo = op_qubits(y);
        if (!((yo.nd | yo.nx | yo.dg) & qb)) continue;
        if (y.kind == FK_GATE && y.cmask == 0 && y.q0 == x.q0) {
            // product X * Y (X applied after Y), complex 2x2 row-major
            double p[8];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) {
                    double re = 0.0, im = 0.0;
                    for (int j = 0; j < 2; ++j) {
                        const double ar = x.m[4 * r + 2 * j], ai = x.m[4 * r + 2 * j + 1];
                        const double br = y.m[4 * j + 2 * c], bi = y.m[4 * j + 2 * c + 1];
                        re += ar * br - ai * bi;
                        im += ar * bi + ai * br;
                    }
                    p[4 * r + 2 * c] = re;
                    p[4 * r + 2 * c + 1] = im;
                }
            uint8_t flags = 0;
            const uint8_t cls = classify(p, &flags);
            if (cls == CLS_GENERIC || cls == CLS_SWAP) return false;
            std::memcpy(y.m, p, sizeof(p));
            y.cls = cls;
            y.flags = flags;
            y.unit = 0;
            // Y's old scalar is already in gscale; this takes X's in
            if (env->normalize) normalize_op(y);
            if (plan_sink && x.id >= 0) merged_ids[y.id].push_back(x.id);
            return true;
        }
        if (blocked_by(xo, [&] {
                Blockers b;
                b.add(yo);
                return b;
            }()))
            return false;
    }
    return false;
}

void QuregImpl::window_drain() {
    while (!win.empty()) window_pass();
}

void QuregImpl::window_pass() {
    if (win.empty()) return;
    const size_t W = win.size();
    std::vector<OpQubits> oq(W);
    uint64_t cand = 0;
    const uint64_t lanes = (uint64_t{1} << kLaneQubits) - 1;
    for (size_t j = 0; j < W; ++j) {
        oq[j] = op_qubits(win[j]);
        cand |= oq[j].need;
    }
    cand &= ~lanes;
    // ops a tile of qubits T admits: one ordered scan
    auto closure = [&](uint64_t T, std::vector<char>* sel) {
        Blockers bl;
        int n = 0;
        for (size_t j = 0; j < W; ++j) {
            const OpQubits& o = oq[j];
            const bool ok = (o.need & ~T) == 0 && !blocked_by(o, bl);
            if (ok) {
                ++n;
            } else {
                bl.add(o);
            }
            if (sel) (*sel)[j] = ok ? 1 : 0;
        }
        return n;
    };
    // high tile qubits: the first op's, then greedy
    uint64_t H = oq[0].need & ~lanes;
    int have = closure(lanes | H, nullptr);
    while (__builtin_popcountll(H) < env->tile_targets) {
        int best = have, bq = -1;
        for (uint64_t c = cand & ~H; c; c &= c - 1) {
            const int q = __builtin_ctzll(c);
            const int n = closure(lanes | H | (uint64_t{1} << q), nullptr);
            if (n > best) {
                best = n;
                bq = q;
            }
        }
        if (bq < 0) break;
        H |= uint64_t{1} << bq;
        have = best;
    }
    std::vector<char> sel(W), taken(W, 0);
    closure(lanes | H, &sel);

    // phases: list scheduling over the selected ops
    discard();
    const size_t cap = static_cast<size_t>(std::min(env->tile_max_ops, kMaxTileOps));
    const int lf = lane_fixed();
    const int maxph = max_phases();
    auto in = [](const std::vector<int>& v, int q) { return std::find(v.begin(), v.end(), q) != v.end(); };
    // register qubits op j still needs in a phase holding R
    auto missing = [&](size_t j, const std::vector<int>& R, int* qs) {
        const FlatOp& op = win[j];
        int k = 0;
        if (op.kind == FK_DEPOL) {
            if (op.q0 >= lf && !in(R, op.q0)) qs[k++] = op.q0;
            if (!in(R, op.q1)) qs[k++] = op.q1;
        } else if (op.kind == FK_GATE && op.cls != CLS_DIAG && op.q0 >= kLaneQubits && !in(R, op.q0)) {
            qs[k++] = op.q0;
        }
        return k;
    };
    // Lane ops (pair targets on lane bits: 4 warp shuffles per amplitude)
    // are taken eagerly by the tile choice (lanes are always in the tile), so
    // without a cap they pile up in the first passes, where the shuffle unit
    // (1 warp instruction / clock / SM) rather than the FP64 pipe bounds the
    // pass; capped per pass they spread out and overlap the FP64 work of the
    // register ops (Env::lane_cap, QGPU_LANE_CAP; 0 = no cap).
    int lane_ops = 0;
    auto shuffles = [&](size_t j, const std::vector<int>& R) {
        const FlatOp& op = win[j];
        if (op.kind == FK_DEPOL) return op.q0 < lf;
        if (op.kind != FK_GATE || op.cls == CLS_DIAG || op.q0 >= kLaneQubits) return false;
        if (op.q0 < lf) return true;
        return !in(R, op.q0) && static_cast<int>(R.size()) >= kPhaseRegBits; // 3, 4 as lane bits
    };
    // Swizzled middle phase (Env::swizzle): when the pass has enough pair ops
    // on the fixed lane qubits 0-2, the first phase holds them back and the
    // second holds qubits 0-2 as register qubits (its lanes 0-2 span three
    // other tile qubits; the shared-memory layouts around it are XOR-swizzled
    // so every access stays conflict-free), so they run without shuffles.
    auto fixed_pair = [&](size_t j) {
        const FlatOp& op = win[j];
        return op.kind == FK_GATE && op.cls != CLS_DIAG && op.q0 < lf;
    };
    bool plan_mid = false;
    if (env->swizzle > 0 && !single && lf == kFixedLaneBits && maxph >= 3) {
        int n = 0;
        for (size_t j = 0; j < W; ++j) n += sel[j] && fixed_pair(j);
        plan_mid = n >= env->swizzle;
    }
    std::vector<size_t> pwin; // window index of each pending op
    for (int attempt = 0;; ++attempt) {
    while (static_cast<int>(phases.size()) < maxph && pending.size() < cap) {
        PhaseState ph;
        ph.op_begin = static_cast<int>(pending.size());
        std::vector<int>& R = ph.regs;
        // (fixed-lane pair ops wait for the middle phase, and after it for
        // the next pass's one rather than shuffling in the last phase:
        // 156.1 vs 156.9 ms per step at lower clocks, profiles/r2/r2sw;
        // QGPU_SWIZZLE_HOLD=0 lets the last phase take them)
        static const bool hold_after = [] {
            const char* v = std::getenv("QGPU_SWIZZLE_HOLD");
            return !v || std::atoi(v) != 0;
        }();
        const bool hold = plan_mid && (phases.empty() || (hold_after && phases.size() >= 2));
        ph.mid = plan_mid && phases.size() == 1;
        if (ph.mid)
            for (int q = 0; q < kFixedLaneBits; ++q) R.push_back(q);
        bool any = false;
        for (;;) {
            bool progress = true;
            while (progress && pending.size() < cap) {
                progress = false;
                Blockers bl;
                for (size_t j = 0; j < W; ++j) {
                    if (!sel[j] || taken[j]) continue;
                    int qs[2];
                    const bool lane = !ph.mid && shuffles(j, R);
                    if (pending.size() < cap && !blocked_by(oq[j], bl) && missing(j, R, qs) == 0 &&
                        !(hold && fixed_pair(j)) && !(lane && env->lane_cap > 0 && lane_ops >= env->lane_cap)) {
                        const FlatOp& op = win[j];
                        if (lane) ++lane_ops;
                        // qubits 3, 4: a register qubit while the phase has
                        // room, else a lane op (as place_tile)
                        if (op.kind == FK_GATE && op.cls != CLS_DIAG && op.q0 >= lf && op.q0 < kLaneQubits &&
                            !in(R, op.q0) && static_cast<int>(R.size()) < kPhaseRegBits)
                            R.push_back(op.q0);
                        pending.push_back(op);
                        pwin.push_back(j);
                        taken[j] = 1;
                        progress = any = true;
                    } else {
                        bl.add(oq[j]);
                    }
                }
            }
            const int room = kPhaseRegBits - static_cast<int>(R.size());
            if (pending.size() >= cap || room <= 0) break;
            // the register qubit that unblocks the most ready ops
            int cnt[64] = {};
            Blockers bl;
            for (size_t j = 0; j < W; ++j) {
                if (!sel[j] || taken[j]) continue;
                if (!blocked_by(oq[j], bl)) {
                    int qs[2];
                    const int k = missing(j, R, qs);
                    if (k > 0 && k <= room)
                        for (int i = 0; i < k; ++i) ++cnt[qs[i]];
                }
                bl.add(oq[j]);
            }
            int bq = -1;
            for (int q = 0; q < 64; ++q)
                if (cnt[q] > 0 && (bq < 0 || cnt[q] > cnt[bq])) bq = q;
            if (bq < 0) break;
            R.push_back(bq);
        }
        if (!any) break;
        phases.push_back(ph);
    }
    // everything the pass could take waited for a middle phase (the window
    // holds only pair ops on qubits 0-2 and what depends on them): plain
    // phases instead
    if (pending.empty() && plan_mid && attempt == 0) {
        plan_mid = false;
        phases.clear();
        pwin.clear();
        lane_ops = 0;
        std::fill(taken.begin(), taken.end(), 0);
        continue;
    }
    break;
    }
    if (pending.empty()) throw DeviceError("internal: reorder scheduler formed an empty pass");
    if (!phases.empty() && phases.back().mid) { // a middle phase must not be last: an empty standard one follows
        PhaseState tail;
        tail.op_begin = static_cast<int>(pending.size());
        phases.push_back(tail);
    }
    // Room for the lane <-> register exchanges launch_tile adds (two per lane
    // qubit with two or more pair ops in a phase, at most one per register
    // bit): the pass's last ops go back to the window if needed (a suffix of
    // a dependency-ordered list: nothing kept depends on them).
    auto xneed = [&]() {
        if (env->exchanges != 1 || plan_mid) return 0; // (2: exchanges only where a pass has room)
        int need = 0;
        for (size_t p = 0; p < phases.size(); ++p) {
            const size_t b = static_cast<size_t>(phases[p].op_begin);
            const size_t e = p + 1 < phases.size() ? static_cast<size_t>(phases[p + 1].op_begin) : pending.size();
            int cnt[kLaneQubits] = {};
            for (size_t k = b; k < e; ++k) {
                const FlatOp& op = pending[k];
                if (op.kind == FK_GATE && op.cls != CLS_DIAG && op.q0 < kLaneQubits && !in(phases[p].regs, op.q0))
                    ++cnt[op.q0];
            }
            int c = 0;
            for (int q = 0; q < kLaneQubits; ++q) c += cnt[q] >= 2;
            need += 2 * std::min(c, kPhaseRegBits);
        }
        return need;
    };
    while (pending.size() > 1 && static_cast<int>(pending.size()) + xneed() > kMaxTileOps) {
        taken[pwin.back()] = 0;
        pwin.pop_back();
        pending.pop_back();
        if (phases.size() > 1 && static_cast<size_t>(phases.back().op_begin) >= pending.size()) phases.pop_back();
    }
    for (const PhaseState& ph : phases)
        for (int q : ph.regs)
            if (q >= kLaneQubits && !in(tile_high, q)) tile_high.push_back(q);
    if (static_cast<int>(tile_high.size()) > kTileHigh)
        throw DeviceError("internal: reorder scheduler exceeded the tile");
    size_t k = 0;
    for (size_t j = 0; j < W; ++j)
        if (!taken[j]) win[k++] = win[j];
    win.resize(k);
    if (!fold_scale() && win.empty()) {
        // the window drains with the scalar unapplied: one elementwise op
        // (any qubit; qubit 0: a lane diagonal) in this pass, or the next
        FlatOp sc;
        sc.kind = FK_GATE;
        sc.cls = CLS_DIAG;
        sc.q0 = 0;
        sc.m[0] = sc.m[6] = gscale_re;
        sc.m[1] = sc.m[7] = gscale_im;
        if (pending.size() < cap) {
            pending.push_back(sc);
            gscale_re = 1.0;
            gscale_im = 0.0;
        } else {
            win.push_back(sc); // carries its own scalar: the pending one is in it
            gscale_re = 1.0;
            gscale_im = 0.0;
        }
    }
    launch_tile();
    discard();
}

void QuregImpl::enqueue(const FlatOp& lop) {
    materialize();
    ++version;
    if (!swaps_on()) {
        enqueue_phys(lop);
        return;
    }
    lq.push_back(lop);
    if (lq.size() >= kSwapWindow) drain(kSwapWindow / 2);
}

// Logical ops -> physical: a pair target (and both qubits of a depolarising
// channel) must be local, so a global one is swapped in first, evicting the
// local qubit next needed furthest ahead in the buffered window; diagonal
// ops, dephasing, collapse and controls work on any position.
// Light-cone drain (the reordering mode): instead of taking the logical queue
// in circuit order — a layered circuit touches every qubit once per layer,
// so the global ones had to be swapped in (and others out) every layer: 34
// swaps per step of the 36-qubit / 8-rank bench circuit — every op that can
// run with the current local qubits and commutes with the ops held back
// before it (op_qubits' rule) is released at once. Only when nothing can run
// does the first held-back op get its global qubits swapped in, evicting the
// local qubit needed furthest ahead in the queue: typically one whose work
// in the queue is done. Dependencies travel one qubit per layer, so the ops
// far from the global qubits run ahead and the 36-qubit circuit needs about
// 3-7 swaps per step (host dry run: qgpuPlanSwapsReorder,
// tests/test_distributed_gloo.py). Results within 1e-12 (commuting ops
// reordered), like the window scheduler downstream.
void QuregImpl::drain_lightcone(size_t count) {
    const size_t target = lq.size() - std::min(count, lq.size()); // ops left queued
    while (lq.size() > target) {
        Blockers bl;
        std::vector<FlatOp> rest;
        rest.reserve(lq.size());
        bool any = false;
        for (const FlatOp& lop : lq) {
            const OpQubits o = op_qubits(lop);
            const bool local = (sp.phys_mask(o.need) >> local_qubits) == 0;
            if (local && !blocked_by(o, bl)) {
                for (uint64_t m = o.need; m; m &= m - 1) sp.touch(__builtin_ctzll(m));
                FlatOp op = lop;
                op.q0 = sp.phys(lop.q0);
                op.q1 = sp.phys(lop.q1);
                op.cmask = sp.phys_mask(lop.cmask);
                enqueue_phys(op);
                any = true;
            } else {
                bl.add(o);
                rest.push_back(lop);
            }
        }
        lq.swap(rest);
        if (lq.size() <= target || any) continue;
        // nothing can run: the first queued op (it has no queued predecessor)
        // needs a global qubit
        std::vector<int> need0(lq.size(), -1), need1(lq.size(), -1);
        for (size_t j = 0; j < lq.size(); ++j) {
            const FlatOp& o = lq[j];
            if (o.kind == FK_GATE && o.cls != CLS_DIAG) need0[j] = o.q0;
            if (o.kind == FK_DEPOL) {
                need0[j] = o.q0;
                need1[j] = o.q1;
            }
        }
        const FlatOp& f = lq.front();
        if (f.kind == FK_GATE && f.cls == CLS_DIAG)
            throw DeviceError("internal: light-cone drain stuck on an op that needs no local qubit");
        auto make_local = [&](int logical, uint64_t busy) {
            const int p = sp.l2p[logical];
            if (p < local_qubits) return;
            uint64_t in_window = 0; // positions the pass window still acts on
            for (const FlatOp& w : win) {
                const OpQubits o = op_qubits(w);
                in_window |= o.nd | o.nx | o.dg | o.need;
            }
            const int v = sp.victim(busy, need0.data() + 1, need1.data() + 1, lq.size() - 1, in_window);
            // Only the released ops on the two traded positions must run
            // before the swap; the rest of the pass window commutes with it
            // (a permutation of other qubits) and stays for fuller passes.
            const uint64_t moved = (uint64_t{1} << p) | (uint64_t{1} << v);
            auto pending_on_moved = [&] {
                for (const FlatOp& w : win) {
                    const OpQubits o = op_qubits(w);
                    if ((o.nd | o.nx | o.dg | o.need) & moved) return true;
                }
                return false;
            };
            while (pending_on_moved()) window_pass();
            run_swap(p, v, /*flush=*/false);
            sp.apply(p, v);
        };
        uint64_t busy0 = 0;
        if (need1[0] >= 0 && sp.l2p[need1[0]] < local_qubits) busy0 = uint64_t{1} << sp.l2p[need1[0]];
        if (need0[0] >= 0) make_local(need0[0], busy0);
        if (need1[0] >= 0) make_local(need1[0], uint64_t{1} << sp.l2p[need0[0]]);
    }
}

void QuregImpl::drain(size_t count) {
    if (reorder_on()) {
        drain_lightcone(count);
        return;
    }
    count = std::min(count, lq.size());
    std::vector<int> need0(lq.size(), -1), need1(lq.size(), -1);
    for (size_t j = 0; j < lq.size(); ++j) {
        const FlatOp& o = lq[j];
        if (o.kind == FK_GATE && o.cls != CLS_DIAG) need0[j] = o.q0;
        if (o.kind == FK_DEPOL) {
            need0[j] = o.q0;
            need1[j] = o.q1;
        }
    }
    for (size_t i = 0; i < count; ++i) {
        const FlatOp& lop = lq[i];
        if (need0[i] >= 0) sp.touch(need0[i]);
        if (need1[i] >= 0) sp.touch(need1[i]);
        auto make_local = [&](int logical, uint64_t busy) {
            const int p = sp.l2p[logical];
            if (p < local_qubits) return;
            const size_t nf = lq.size() - i - 1;
            const int v = sp.victim(busy, need0.data() + i + 1, need1.data() + i + 1, nf);
            run_swap(p, v);
            sp.apply(p, v);
        };
        // a channel's second qubit that is already local must not be evicted
        // to make room for the first (it would be swapped straight back)
        uint64_t busy0 = 0;
        if (need1[i] >= 0 && sp.l2p[need1[i]] < local_qubits) busy0 = uint64_t{1} << sp.l2p[need1[i]];
        if (need0[i] >= 0) make_local(need0[i], busy0);
        if (need1[i] >= 0) make_local(need1[i], uint64_t{1} << sp.l2p[need0[i]]);
        FlatOp op = lop;
        op.q0 = sp.phys(lop.q0);
        op.q1 = sp.phys(lop.q1);
        op.cmask = sp.phys_mask(lop.cmask);
        enqueue_phys(op);
    }
    lq.erase(lq.begin(), lq.begin() + static_cast<std::ptrdiff_t>(count));
}

void QuregImpl::enqueue_phys(const FlatOp& op) {
    const bool pair = op.kind == FK_GATE && op.cls != CLS_DIAG;
    if (reorder_on()) {
        // ops a tile pass can take wait in the window; anything else
        // (exchange gates, unfusable channels) runs after the window drains
        const bool tileable = op.kind == FK_DEPOL
                                  ? op.q1 >= lane_fixed() && op.q0 < local_qubits && op.q1 < local_qubits
                                  : !(pair && op.q0 >= local_qubits);
        if (tileable) {
            if (env->merge && merge_into_window(op)) return;
            win.push_back(op);
            if (env->normalize) normalize_op(win.back());
            if (static_cast<int>(win.size()) >= env->window) window_pass();
            return;
        }
        window_drain();
    }
    if (op.kind == FK_DEPOL) {
        // fused into the tile pass when both qubits can be register qubits
        // of a phase (not lane-only qubits 0-2); else its own pass
        // (t on a fixed lane bit: the lane variant, TC_DEPOL_LANE)
        const bool fusable = use_tile() && env->fusion_mode == 0 && op.q1 >= lane_fixed() &&
                             op.q0 < local_qubits && op.q1 < local_qubits;
        if (!fusable) {
            flush_pass();
            run_depol(op);
            return;
        }
        if (!place_tile_depol(op)) {
            flush_pass();
            place_tile_depol(op);
        }
        if (static_cast<int>(pending.size()) >= std::min(env->tile_max_ops, kMaxTileOps)) flush_pass();
        return;
    }
    if (pair && op.q0 >= local_qubits) {
        flush_pass();
        run_exchange_gate(op);
        return;
    }
    // states too small to tile run one kernel per op in single precision (the
    // register-only small-state pass is instantiated for double only)
    if (env->fusion_mode == 2 || pass_H() < 1 || (single && !use_tile())) {
        flush_pass();
        run_simple(op);
        ++passes;
        return;
    }
    if (use_tile()) {
        if (!place_tile(op, pair)) {
            flush_pass();
            place_tile(op, pair);
        }
        if (env->fusion_mode == 1 ||
            static_cast<int>(pending.size()) >= std::min(env->tile_max_ops, kMaxTileOps))
            flush_pass();
        return;
    }
    if (pair && op.q0 >= kLaneQubits &&
        std::find(regs.begin(), regs.end(), op.q0) == regs.end()) {
        if (static_cast<int>(regs.size()) >= pass_H()) flush_pass();
        regs.push_back(op.q0);
    }
    pending.push_back(op);
    if (env->fusion_mode == 1 || static_cast<int>(pending.size()) >= env->max_ops) flush_pass();
}

void QuregImpl::flush() {
    materialize();
    if (!lq.empty()) drain(lq.size());
    flush_pass();
}

void QuregImpl::defer_collapse(const FlatOp& op) {
    ++version;
    deferred.push_back(op);
}

void QuregImpl::materialize() {
    if (deferred.empty()) return;
    std::vector<FlatOp> d;
    d.swap(deferred);
    for (const FlatOp& op : d) enqueue(op);
}

void QuregImpl::flush_pass() {
    window_drain();
    if (!pending.empty()) {
        if (use_tile() && env->fusion_mode != 2)
            launch_tile();
        else
            launch_fused();
    }
    discard();
}

// QGPU_PASS_STATS=1: histogram of tile-pass handler codes and phase counts,
// printed at exit (scheduler / kernel tuning aid; off by default).
namespace {
struct PassStats {
    uint64_t passes = 0, phases = 0, ops = 0, outer = 0, skipping = 0;
    uint64_t code[64] = {};
    ~PassStats() {
        if (!passes) return;
        std::fprintf(stderr, "[qgpu pass stats] passes %llu, phases/pass %.2f, ops/pass %.2f, outer-controlled %.1f%%, "
                     "tile-skipping passes %llu\n",
                     (unsigned long long)passes, double(phases) / passes, double(ops) / passes,
                     100.0 * double(outer) / double(ops ? ops : 1), (unsigned long long)skipping);
        for (int c = 0; c < 64; ++c)
            if (code[c])
                std::fprintf(stderr, "  code %2d: %6.2f per pass\n", c, double(code[c]) / passes);
    }
};
PassStats g_pass_stats;
} // namespace

bool pass_stats_enabled() {
    static const bool on = std::getenv("QGPU_PASS_STATS") != nullptr;
    return on;
}

void record_pass_stats(const TileParams& P) {
    const int nops = P.phases[P.num_phases - 1].op_end;
    ++g_pass_stats.passes;
    if (P.skip_ones) ++g_pass_stats.skipping;
    g_pass_stats.phases += P.num_phases;
    g_pass_stats.ops += nops;
    for (int k = 0; k < nops; ++k) {
        ++g_pass_stats.code[P.ops[k].hdr & 63];
        if (P.ops[k].outer_cmask) ++g_pass_stats.outer;
    }
}

// Profile record of a tile pass: ops (bits 0-7), phases (8-15) and a model
// of the FP64 instructions per amplitude x 4 (16-31) — the reference's fma
// chain per handler class (8 for a generic 2x2 row pair, 4 for real /
// Rx-class rows and diagonals, 0 for swaps), halved per control outside the
// tile (those tiles skip the op) and for a == 1 diagonals on warp / outer
// qubits (the identity side copies). bench.py turns it into the pass's FP64
// time bound beside its HBM bound.
int pass_profile_info(const TileParams& P) {
    const int nops = P.phases[P.num_phases - 1].op_end;
    double fp = 0.0;
    for (int k = 0; k < nops; ++k) {
        const uint64_t h = P.ops[k].hdr;
        const int code = static_cast<int>(h & 63);
        const uint32_t flags = (h >> 6) & 15u;
        double f;
        const uint32_t un = static_cast<uint32_t>((h >> 40) & 0xff);
        auto u = [&](int k) { return (un >> (2 * k)) & 3u; };
        if (code < TC_REG + 4) { // 2x2 on a register bit, by class row
            const int row = code - TC_REG;
            f = row == 0 ? 8.0 : row == 3 ? 0.0 : 4.0;
            if (row == 1 || row == 2) // unit coefficients: one FMA (or add) per component
                f = ((u(0) || u(1)) ? 1.0 : 2.0) + ((u(2) || u(3)) ? 1.0 : 2.0);
        } else if (code < TC_REG_SEL + 2) {
            f = code == TC_REG_SEL ? 8.0 : 0.0;
        } else if (code == TC_LANE_GENERIC || code == TC_LANE_SEL_GENERIC) {
            f = 8.0;
        } else if (code == TC_LANE_REAL || code == TC_LANE_RX) {
            // a unit M (m00, m11) or T (m01, m10) on both rows: one FMA per component (lin2)
            const bool uni = (u(1) && u(2)) || (u(0) && u(3));
            f = uni ? 2.0 : 4.0;
        } else if (code == TC_LANE_XCHG) {
            f = 0.0;
        } else if (code == TC_LANE_SWAP || code == TC_LANE_SEL_SWAP) {
            f = 0.0;
        } else if (code == TC_DIAG_REG_D || code == TC_DIAG_REG_D_SEL) {
            f = 2.0; // only the bit-1 half
        } else if (code == TC_DIAG_UNIFORM || code == TC_DIAG_UNIFORM_SEL) {
            f = (flags & (DF_A_ONE | DF_D_ONE)) ? 2.0 : 4.0;
        } else if (code == TC_DIAG_LANE && u(0) == 1) {
            f = 2.0; // symmetric form: two FMAs
        } else if (code == TC_DEPHASE || code == TC_COLLAPSE) {
            f = 2.0;
        } else if (code == TC_DEPOL || code == TC_DEPOL_LANE) {
            f = 3.0;
        } else {
            f = 4.0; // the other diagonals
        }
        f *= std::ldexp(1.0, -__builtin_popcountll(P.ops[k].outer_cmask));
        fp += f;
    }
    const int fp4 = std::min(32767, static_cast<int>(fp * 4.0 + 0.5));
    return nops | (P.num_phases << 8) | (fp4 << 16);
}

void QuregImpl::launch_tile() {
    if (plan_sink) {
        PlannedPass pp;
        std::vector<int> at(pending.size() + 1, 0); // index into ids of each pending op
        for (size_t k = 0; k < pending.size(); ++k) {
            at[k] = static_cast<int>(pp.ids.size());
            pp.ids.push_back(pending[k].id);
            auto it = merged_ids.find(pending[k].id);
            if (it != merged_ids.end())
                for (int id : it->second) pp.ids.push_back(id);
        }
        at[pending.size()] = static_cast<int>(pp.ids.size());
        for (const PhaseState& ph : phases) pp.phase_begin.push_back(at[ph.op_begin]);
        plan_sink->push_back(std::move(pp));
        // QGPU_PLAN_JIT_DUMP=<dir>: dry runs also build the pass parameters
        // and write each pass's generated JIT program there (offline SASS
        // inspection: tools/jit_offline.py)
        static const char* dump_dir = std::getenv("QGPU_PLAN_JIT_DUMP");
        if (!dump_dir) {
            ++passes;
            return;
        }
    }
    // The tile's high qubits: the pass's pair targets, topped up with the
    // lowest unused local qubits (qubits 5, 6, 7 let a warp's last-phase
    // segments merge into longer bulk copies, see P.fin_run).
    std::vector<int> high = tile_high;
    // qubits every op needs at 1 (common controls, diagonal targets with
    // a == 1) are topped up last: outside the tile they let the pass skip
    // every tile where they are 0 (TileParams.skip_ones)
    uint64_t need = ~uint64_t{0};
    for (const FlatOp& op : pending) {
        uint64_t m = op.kind == FK_GATE ? op.cmask : 0;
        if (op.kind == FK_GATE && op.cls == CLS_DIAG && (op.flags & DF_A_ONE)) m |= uint64_t{1} << op.q0;
        need &= m;
    }
    for (int pass = 0; pass < 2; ++pass)
        for (int q = kLaneQubits; static_cast<int>(high.size()) < kTileHigh && q < local_qubits; ++q)
            if (std::find(high.begin(), high.end(), q) == high.end() && (pass == 1 || !((need >> q) & 1)))
                high.push_back(q);
    std::sort(high.begin(), high.end());
    auto tbit = [&](int q) -> int { // tile bit of a local qubit, -1 if outside
        if (q >= 0 && q < kLaneQubits) return q;
        for (int j = 0; j < kTileHigh; ++j)
            if (high[j] == q) return kLaneQubits + j;
        return -1;
    };

    TileParams P;
    std::memset(&P, 0, sizeof(P));
    P.num_tiles = uint64_t{1} << (local_qubits - kTileQubits);
    P.single = single ? 1 : 0;
    P.fast = env->order == 1 ? 1 : 0; // tolerance-mode handlers with the reordering schedule
    P.num_phases = static_cast<int>(phases.size());
    for (int j = 0; j < kTileHigh; ++j) P.high_pos[j] = high[j];
    for (int s = 0; s < (1 << kTileHigh); ++s) {
        uint64_t off = 0;
        for (int j = 0; j < kTileHigh; ++j)
            if ((s >> j) & 1) off |= uint64_t{1} << high[j];
        P.seg_off[s] = off;
    }
    // Per phase: register bits (the phase's targets, topped up), lane bits 3-4
    // and warp bits (the rest of tile bits 3..11). Layouts are chosen so that
    // consecutive phases share as many warp bits as possible, at the same
    // (top) warp-index positions: data then only moves within groups of
    // 2^(WB - c) warps, which synchronise on a named barrier instead of the
    // whole CTA (c = shared bits; kernel: TilePhase.sync_bits).
    const size_t nph = phases.size();
    std::vector<std::vector<int>> RB(nph), LB(nph), WBv(nph), KB(nph); // KB: a middle phase's lanes 0-2
    auto has = [](const std::vector<int>& v, int t) { return std::find(v.begin(), v.end(), t) != v.end(); };
    for (size_t p = 0; p < nph; ++p)
        for (int q : phases[p].regs) RB[p].push_back(tbit(q));
    for (size_t p = nph; p-- > 0;) {
        std::vector<int> pref; // bits better kept off this phase's warp bits
        if (p + 1 < nph) {
            for (int t : RB[p + 1]) pref.push_back(t);
            for (int t : LB[p + 1]) pref.push_back(t);
        }
        const bool last = p + 1 == nph;
        // top up the register bits: first from `pref`, then the lowest free
        for (int t : pref)
            if (static_cast<int>(RB[p].size()) < kPhaseRegBits && t >= kLaneQubits && !has(RB[p], t))
                RB[p].push_back(t);
        for (int t = kLaneQubits; t < kTileQubits && static_cast<int>(RB[p].size()) < kPhaseRegBits; ++t)
            if (!has(RB[p], t)) RB[p].push_back(t);
        // lane bits 3-4: in the last phase tile bits 3, 4 unless registers
        // (tile bits 0-4 are never warp bits there: per-warp segments);
        // earlier phases prefer bits of `pref`
        // single precision: tile bit 3 is always lane bit 3 (8-byte
        // amplitudes: lanes must span 16 consecutive amplitudes to cover the
        // 32 shared-memory banks; place_tile never makes qubit 3 a register)
        if (pin_lane3()) LB[p].push_back(3);
        if (last) {
            for (int t = kFixedLaneBits; t < kTileQubits && LB[p].size() < 2; ++t)
                if (!has(RB[p], t) && !has(LB[p], t)) LB[p].push_back(t);
        } else {
            // qubits 3, 4 targeted by this phase's pair ops (as lane ops,
            // place_tile) must stay lane bits
            const int begin = phases[p].op_begin;
            const int end = phases[p + 1].op_begin;
            for (int k = begin; k < end; ++k) {
                const FlatOp& op = pending[k];
                const bool pair = op.kind == FK_GATE && op.cls != CLS_DIAG;
                if (pair && op.q0 >= kFixedLaneBits && op.q0 < kLaneQubits && !has(RB[p], op.q0) &&
                    !has(LB[p], op.q0))
                    LB[p].push_back(op.q0);
            }
            for (int t : pref) // (a middle phase's registers include tile bits 0-2: never lane bits 3-4)
                if (LB[p].size() < 2 && t >= kFixedLaneBits && !has(RB[p], t) && !has(LB[p], t)) LB[p].push_back(t);
            for (int t = kFixedLaneBits; t < kTileQubits && LB[p].size() < 2; ++t)
                if (!has(RB[p], t) && !has(LB[p], t)) LB[p].push_back(t);
        }
        if (phases[p].mid) // lanes 0-2: three other tile bits (qubits 0-2 are registers here)
            for (int t = kTileQubits - 1; t >= kFixedLaneBits && KB[p].size() < 3; --t)
                if (!has(RB[p], t) && !has(LB[p], t)) KB[p].push_back(t);
        for (int t = kFixedLaneBits; t < kTileQubits; ++t)
            if (!has(RB[p], t) && !has(LB[p], t) && !has(KB[p], t)) WBv[p].push_back(t);
    }
    // order warp bits: bits shared with the next phase on top (same order)
    std::vector<int> sync_bits(nph, 0);
    for (size_t p = 0; p + 1 < nph; ++p) {
        std::vector<int> common;
        for (int t : WBv[p])
            if (has(WBv[p + 1], t)) common.push_back(t);
        auto reorder = [&](std::vector<int>& wb, bool keep_top) {
            std::vector<int> rest;
            for (int t : wb)
                if (!has(common, t)) rest.push_back(t);
            std::vector<int> out = rest;
            for (int t : common) out.push_back(t);
            if (keep_top) {
                // the next phase may already be ordered for its own next
                // transition: only sync in groups if the positions agree
                return;
            }
            wb = out;
        };
        reorder(WBv[p], false);
        // the next phase: put the common bits at the same top positions
        // unless that breaks its own (already fixed) order — phases are
        // processed front to back, so only the first transition of a
        // 3+-phase pass could be affected; check positions explicitly
        std::vector<int> rest;
        for (int t : WBv[p + 1])
            if (!has(common, t)) rest.push_back(t);
        std::vector<int> nb = rest;
        for (int t : common) nb.push_back(t);
        WBv[p + 1] = nb;
        (void)reorder;
    }
    for (size_t p = 1; p < nph; ++p) {
        int c = 0;
        while (c < kTileWarpBits &&
               WBv[p][kTileWarpBits - 1 - c] == WBv[p - 1][kTileWarpBits - 1 - c])
            ++c;
        sync_bits[p] = c;
    }
    // named barrier IDs (per tile group: relative IDs 1 .. kBarIdsPerGroup-1,
    // qgpu_device.h): each transition its own range of 2^c IDs (a shared ID
    // let a lagging warp of one transition complete another's barrier, and
    // mixed thread counts trap); transitions that do not fit sync the whole
    // group
    std::vector<int> bar_base(nph, 0);
    {
        int next_id = 1;
        for (size_t p = 1; p < nph; ++p) {
            const int c = sync_bits[p];
            if (c == 0 || c >= kTileWarpBits) continue; // group barrier / warp sync
            if (next_id + (1 << c) > kBarIdsPerGroup) {
                sync_bits[p] = 0;
                continue;
            }
            bar_base[p] = next_id;
            next_id += 1 << c;
        }
    }
    // Renumber the high tile bits so the last phase's non-warp high bits sit
    // at tile bits 5..7 in ascending qubit order: each warp's 8 last-phase
    // segments are then contiguous in shared memory, and whenever those
    // qubits are 5, 6, 7 they are contiguous in HBM too, so the warp moves
    // them in fewer, larger bulk copies (P.fin_run). Only names change: the
    // layouts above are remapped, not recomputed.
    {
        const std::vector<int>& wl = WBv[nph - 1];
        std::vector<int> order; // new tile bit 5 + k := old tile bit order[k]
        for (int t = kLaneQubits; t < kTileQubits; ++t)
            if (!has(wl, t)) order.push_back(t);
        for (int t = kLaneQubits; t < kTileQubits; ++t)
            if (has(wl, t)) order.push_back(t);
        std::vector<int> remap(kTileQubits);
        for (int t = 0; t < kLaneQubits; ++t) remap[t] = t;
        std::vector<int> nh(kTileHigh);
        for (int k = 0; k < kTileHigh; ++k) {
            remap[order[k]] = kLaneQubits + k;
            nh[k] = high[order[k] - kLaneQubits];
        }
        high = nh;
        for (size_t p = 0; p < nph; ++p)
            for (auto* v : {&RB[p], &LB[p], &WBv[p], &KB[p]})
                for (int& t : *v) t = remap[t];
        for (int j = 0; j < kTileHigh; ++j) P.high_pos[j] = high[j];
        {
            std::vector<int> hs = high;
            std::sort(hs.begin(), hs.end());
            for (int j = 0; j < kTileHigh; ++j) P.high_sorted[j] = hs[j];
        }
        for (int sg = 0; sg < (1 << kTileHigh); ++sg) {
            uint64_t off = 0;
            for (int j = 0; j < kTileHigh; ++j)
                if ((sg >> j) & 1) off |= uint64_t{1} << high[j];
            P.seg_off[sg] = off;
        }
        int run = 0; // runs of 2^run segments contiguous in HBM
        while (run < kTileHigh - kTileWarpBits && high[run] == kLaneQubits + run) ++run;
        P.fin_run = run;
    }
    // Lane <-> register exchanges for one phase's ops [begin, end): a lane
    // qubit (a tile bit on lane bits 0-4) with two or more pair ops in the
    // phase moves to a register bit J for the run from its first to its last
    // pair op, and back after it (TC_LANE_XCHG: half a lane op's shuffles
    // each), so those ops run as register ops instead of shuffle-bound lane
    // ops. J's qubit must have no pair op or depolarising channel inside the
    // run (it sits on the lane bit meanwhile; its diagonal ops and controls
    // work there). Returns the phase's emitted sequence: pending indices, and
    // exchanges encoded as -1 - (b * kPhaseRegBits + J). `room`: ops the pass
    // can still take (two per exchange). Pure moves: exact in both modes.
    auto plan_exchanges = [&](int begin, int end, const int* lane_t, const int* reg_t, int room) {
        auto pair_t = [&](const FlatOp& op) { // the tile bit an op pairs on (-1: none)
            return op.kind == FK_GATE && op.cls != CLS_DIAG ? tbit(op.q0) : -1;
        };
        struct X {
            int b, J, first, last;
        };
        std::vector<X> xs;
        bool depol = false;
        for (int k = begin; k < end; ++k) depol |= pending[k].kind == FK_DEPOL;
        if (env->exchanges && room >= 2 && !depol) {
            // Greedy over intervals: lane bit b's qubit sits on register bit J
            // from its use u_i to its use u_j (both pair ops on it), while J's
            // qubit waits on lane bit b (its pair ops there become lane ops).
            // Benefit in lane ops: (j - i + 1) - (J's pair ops inside) - 1
            // (the two exchanges: half a lane op each). Intervals sharing a
            // lane bit or a register bit must not overlap.
            std::vector<int> uses[kLaneQubits], busy[kPhaseRegBits];
            for (int k = begin; k < end; ++k) {
                const int t = pair_t(pending[k]);
                for (int b = 0; b < kLaneQubits; ++b)
                    if (t == lane_t[b]) uses[b].push_back(k);
                for (int J = 0; J < kPhaseRegBits; ++J)
                    if (t == reg_t[J]) busy[J].push_back(k);
            }
            auto overlaps = [](const X& x, int f, int l) { return !(x.last < f || l < x.first); };
            for (;;) {
                int best = 0;
                X bx{-1, -1, -1, -1};
                for (int b = 0; b < kLaneQubits; ++b) {
                    const std::vector<int>& u = uses[b];
                    for (size_t i = 0; i < u.size(); ++i)
                        for (size_t j = i + 1; j < u.size(); ++j) {
                            bool lane_free = true;
                            for (const X& x : xs)
                                if (x.b == b && overlaps(x, u[i], u[j])) lane_free = false;
                            if (!lane_free) break; // (longer runs overlap too)
                            for (int J = 0; J < kPhaseRegBits; ++J) {
                                bool free = true;
                                for (const X& x : xs)
                                    if (x.J == J && overlaps(x, u[i], u[j])) free = false;
                                if (!free) continue;
                                int inside = 0;
                                for (int k : busy[J]) inside += k > u[i] && k < u[j];
                                const int gain = static_cast<int>(j - i + 1) - inside - 1;
                                if (gain > best) {
                                    best = gain;
                                    bx = X{b, J, u[i], u[j]};
                                }
                            }
                        }
                }
                if (best <= 0 || room < 2) break;
                xs.push_back(bx);
                room -= 2;
            }
        }
        std::vector<int> seq;
        for (int k = begin; k < end; ++k) {
            for (const X& x : xs)
                if (x.first == k) seq.push_back(-1 - (x.b * kPhaseRegBits + x.J));
            seq.push_back(k);
            for (const X& x : xs)
                if (x.last == k) seq.push_back(-1 - (x.b * kPhaseRegBits + x.J));
        }
        return seq;
    };
    // Swizzled passes (a middle phase, PhaseState::mid): the shared-memory
    // position of tile index x in the buffers written by the first and the
    // middle phase is x ^ spread(x), spread() moving the middle phase's lane
    // tile bits K[0..2] to bits 0-2. A quarter-warp then hits 8 distinct
    // 16-byte bank groups both where its lanes span tile bits 0-2 (the first
    // and last phases) and where they span K (the middle phase); the TMA fill
    // read by the first phase stays linear. Positions are linear in x, so
    // each phase's per-part offsets combine by XOR (TilePhase.swz).
    std::vector<int> key;
    for (size_t p = 0; p < nph; ++p)
        if (phases[p].mid) key = KB[p];
    const bool swz = !key.empty();
    auto pos = [&](uint32_t x, bool keyed) {
        if (!keyed) return x;
        uint32_t sp3 = 0;
        for (int j = 0; j < 3; ++j) sp3 |= ((x >> key[j]) & 1u) << j;
        return x ^ sp3;
    };
    int ko = 0, xchg_used = 0; // emitted ops, exchanges among them
    for (size_t p = 0; p < phases.size(); ++p) {
        TilePhase& Q = P.phases[p];
        const std::vector<int>& rb = RB[p];
        const std::vector<int>& lb = LB[p];
        const std::vector<int>& wb = WBv[p];
        Q.sync_bits = static_cast<uint16_t>(sync_bits[p]);
        Q.bar_base = static_cast<uint16_t>(bar_base[p]);
        const bool in_keyed = swz && p > 0, out_keyed = swz && p + 1 < nph;
        for (int i = 0; i < (1 << kPhaseRegBits); ++i) {
            uint32_t off = 0;
            for (int j = 0; j < kPhaseRegBits; ++j)
                if ((i >> j) & 1) off |= 1u << rb[j];
            Q.reg_off[i] = static_cast<uint16_t>(pos(off, in_keyed));
            Q.reg_out[i] = static_cast<uint16_t>(pos(off, out_keyed));
        }
        for (int w = 0; w < (1 << kTileWarpBits); ++w) {
            uint32_t off = 0;
            for (int j = 0; j < kTileWarpBits; ++j)
                if ((w >> j) & 1) off |= 1u << wb[j];
            Q.warp_off[w] = static_cast<uint16_t>(pos(off, in_keyed));
            Q.warp_out[w] = static_cast<uint16_t>(pos(off, out_keyed));
        }
        for (int j = 0; j < 2; ++j) Q.lane_off[j] = static_cast<uint16_t>(1u << lb[j]);
        // tile bits on lane bits 0-4
        const int lt[kLaneQubits] = {phases[p].mid ? KB[p][0] : 0, phases[p].mid ? KB[p][1] : 1,
                                     phases[p].mid ? KB[p][2] : 2, lb[0], lb[1]};
        Q.swz = swz ? 1 : 0;
        { // every tile bit exactly once on a lane, register or warp bit of this phase
            uint32_t seen = 0;
            auto claim = [&](int t) {
                if (t < 0 || t >= kTileQubits || ((seen >> t) & 1u))
                    throw DeviceError("internal: tile layout maps a tile bit twice");
                seen |= 1u << t;
            };
            for (int t : lt) claim(t);
            for (int j = 0; j < kPhaseRegBits; ++j) claim(rb[j]);
            for (int j = 0; j < kTileWarpBits; ++j) claim(wb[j]);
        }
        for (int j = 0; j < kLaneQubits; ++j) {
            Q.lane_in[j] = static_cast<uint16_t>(pos(1u << lt[j], in_keyed));
            Q.lane_out[j] = static_cast<uint16_t>(pos(1u << lt[j], out_keyed));
        }
        auto gbit = [&](int t) -> uint64_t {
            return t < kLaneQubits ? uint64_t{1} << t : uint64_t{1} << high[t - kLaneQubits];
        };
        if (p == 0) {
            // first phase (LDG mode loads it from HBM): the same offsets
            for (int i = 0; i < (1 << kPhaseRegBits); ++i) {
                uint64_t g = 0;
                for (int j = 0; j < kPhaseRegBits; ++j)
                    if ((i >> j) & 1) g |= gbit(rb[j]);
                P.first_greg[i] = g;
            }
            for (int w = 0; w < (1 << kTileWarpBits); ++w) {
                uint64_t g = 0;
                for (int j = 0; j < kTileWarpBits; ++j)
                    if ((w >> j) & 1) g |= gbit(wb[j]);
                P.first_gwarp[w] = g;
            }
            for (int j = 0; j < 2; ++j) P.first_glane[j] = gbit(lb[j]);
        }
        if (p + 1 == phases.size()) {
            // last phase: HBM offsets of its registers, warps and lane bits
            for (int i = 0; i < (1 << kPhaseRegBits); ++i) {
                uint64_t g = 0;
                for (int j = 0; j < kPhaseRegBits; ++j)
                    if ((i >> j) & 1) g |= gbit(rb[j]);
                P.fin_greg[i] = g;
            }
            for (int w = 0; w < (1 << kTileWarpBits); ++w) {
                uint64_t g = 0;
                for (int j = 0; j < kTileWarpBits; ++j)
                    if ((w >> j) & 1) g |= gbit(wb[j]);
                P.fin_gwarp[w] = g;
            }
            for (int j = 0; j < 2; ++j) P.fin_glane[j] = gbit(lb[j]);
        }
        if (p + 1 == phases.size()) {
            // last phase: warp w owns the segments whose warp bits are w
            // (tile bits 0-4 are lane or register bits, never warp bits)
            std::vector<int> free_hi;
            for (int t = kLaneQubits; t < kTileQubits; ++t)
                if (std::find(wb.begin(), wb.end(), t) == wb.end()) free_hi.push_back(t - kLaneQubits);
            for (int w = 0; w < (1 << kTileWarpBits); ++w) {
                uint32_t base = 0;
                for (int j = 0; j < kTileWarpBits; ++j)
                    if ((w >> j) & 1) base |= 1u << (wb[j] - kLaneQubits);
                for (int i = 0; i < (1 << (kTileHigh - kTileWarpBits)); ++i) {
                    uint32_t sg = base;
                    for (size_t j = 0; j < free_hi.size(); ++j)
                        if ((i >> j) & 1) sg |= 1u << free_hi[j];
                    P.fin_seg[w][i] = static_cast<uint8_t>(sg);
                }
            }
        }
        const int begin = phases[p].op_begin;
        const int end = p + 1 < phases.size() ? phases[p + 1].op_begin : static_cast<int>(pending.size());
        // Where each tile bit sits while the phase's ops run: lane bits 0-4
        // and register bits, updated by lane <-> register exchanges
        // (plan_exchanges: a run of pair ops on a lane qubit runs on a
        // register bit between two exchanges instead of as shuffle ops).
        int cur_lane[kLaneQubits] = {lt[0], lt[1], lt[2], lt[3], lt[4]};
        int cur_reg[kPhaseRegBits];
        for (int j = 0; j < kPhaseRegBits; ++j) cur_reg[j] = rb[j];
        const int xroom = swz ? 0 : kMaxTileOps - static_cast<int>(pending.size()) - xchg_used;
        const std::vector<int> seq = plan_exchanges(begin, end, cur_lane, cur_reg, xroom);
        Q.op_begin = static_cast<uint16_t>(ko);
        auto loc = [&](int q, uint8_t* kind, uint8_t* pos) {
            const int t = tbit(q);
            *kind = TL_OUTER;
            *pos = static_cast<uint8_t>(q < 0 ? 0 : q);
            if (q < 0 || t < 0) return;
            for (int j = 0; j < kLaneQubits; ++j)
                if (cur_lane[j] == t) {
                    *kind = TL_LANE;
                    *pos = static_cast<uint8_t>(j);
                    return;
                }
            for (int j = 0; j < kPhaseRegBits; ++j)
                if (cur_reg[j] == t) {
                    *kind = TL_REG;
                    *pos = static_cast<uint8_t>(j);
                    return;
                }
            for (int j = 0; j < kTileWarpBits; ++j)
                if (wb[j] == t) {
                    *kind = TL_WARP;
                    *pos = static_cast<uint8_t>(j);
                    return;
                }
        };
        for (const int e : seq) {
            TileOp& to = P.ops[ko++];
            if (e < 0) { // exchange: lane bit b <-> register bit J (encoded -1 - (b * 4 + J))
                const int b = (-1 - e) / kPhaseRegBits, J = (-1 - e) % kPhaseRegBits;
                std::swap(cur_lane[b], cur_reg[J]);
                ++xchg_used;
                if (!plan_sink) ++g_lane_exchanges;
                to.hdr = tile_hdr(TC_LANE_XCHG, 0, 0, TL_LANE, static_cast<uint32_t>(b), TL_REG,
                                  static_cast<uint32_t>(J), 0, 0, 0);
                to.outer_cmask = 0;
                std::memset(to.m, 0, sizeof(to.m));
                continue;
            }
            const FlatOp& op = pending[e];
            const uint32_t flags = op.kind == FK_COLLAPSE ? (op.q1 >= 0 ? 1 : 0) : op.flags;
            uint8_t q0k = 0, q0p = 0, q1k = 0, q1p = 0;
            loc(op.q0, &q0k, &q0p);
            loc(op.q1, &q1k, &q1p);
            uint32_t lane_cm = 0, reg_cm = 0, warp_cm = 0;
            uint64_t outer = op.cmask;
            for (int q = 0; q < local_qubits; ++q) {
                if (!((op.cmask >> q) & 1)) continue;
                uint8_t ck = 0, cp = 0;
                loc(q, &ck, &cp);
                if (ck == TL_OUTER) continue;
                outer &= ~(uint64_t{1} << q);
                if (ck == TL_LANE) lane_cm |= 1u << cp;
                if (ck == TL_REG) reg_cm |= 1u << cp;
                if (ck == TL_WARP) warp_cm |= 1u << cp;
            }
            // resolve the kernel's handler (qgpu_device.h: TileCode); lane,
            // register and warp controls need the per-element predicate (SEL
            // codes), outer controls skip the op per tile
            const bool ctrl = lane_cm != 0 || reg_cm != 0 || warp_cm != 0;
            uint32_t code;
            if (op.kind == FK_DEPOL && q0k == TL_LANE && q1k == TL_REG) {
                code = TC_DEPOL_LANE;
            } else if (op.kind == FK_DEPOL) {
                if (q0k != TL_REG || q1k != TL_REG)
                    throw DeviceError("internal: a fused depolarising channel needs register qubits");
                if (q0p > q1p) std::swap(q0p, q1p); // (symmetric in its two qubits)
                code = TC_DEPOL;
            } else if (op.kind == FK_DEPHASE) {
                code = TC_DEPHASE;
            } else if (op.kind == FK_COLLAPSE) {
                code = TC_COLLAPSE;
            } else if (op.cls == CLS_DIAG) {
                if (q0k == TL_REG) {
                    // a == 1 exactly: the low side is the identity (a * v
                    // with a = 1 + 0i rounds to v), leave it alone
                    const bool d_only = (op.flags & DF_A_ONE) != 0;
                    code = ctrl ? (d_only ? TC_DIAG_REG_D_SEL : TC_DIAG_REG_SEL)
                                : (d_only ? TC_DIAG_REG_D : TC_DIAG_REG);
                } else if (q0k == TL_LANE) {
                    code = ctrl ? TC_DIAG_LANE_SEL : TC_DIAG_LANE;
                } else {
                    code = ctrl ? TC_DIAG_UNIFORM_SEL : TC_DIAG_UNIFORM;
                }
            } else if (q0k == TL_LANE) {
                if (!ctrl)
                    code = op.cls == CLS_SWAP                    ? TC_LANE_SWAP
                           : op.cls == CLS_REAL                  ? TC_LANE_REAL
                           : op.cls == CLS_RX && P.fast ? TC_LANE_RX
                                                                 : TC_LANE_GENERIC;
                else
                    code = op.cls == CLS_SWAP ? TC_LANE_SEL_SWAP : TC_LANE_SEL_GENERIC;
            } else { // register bit
                if (!ctrl) {
                    const uint32_t row = op.cls == CLS_REAL ? 1 : op.cls == CLS_RX ? 2 : op.cls == CLS_SWAP ? 3 : 0;
                    code = TC_REG + row;
                } else {
                    code = TC_REG_SEL + (op.cls == CLS_SWAP ? 1 : 0);
                }
            }
            to.hdr = tile_hdr(code, flags, op.outcome, q0k, q0p, q1k, q1p, lane_cm, reg_cm, warp_cm);
            if (P.fast) to.hdr |= static_cast<uint64_t>(op.unit) << 40; // unit coefficients
            // a diagonal gate with a == 1 exactly (Z, S, T, phase shifts)
            // on a qubit outside the tile is the identity wherever that bit
            // is 0: a control on it, so those tiles skip the op
            if (op.kind == FK_GATE && op.cls == CLS_DIAG && q0k == TL_OUTER && (op.flags & DF_A_ONE))
                outer |= uint64_t{1} << op.q0;
            to.outer_cmask = outer;
            if (outer) P.any_outer = 1;
            std::memcpy(to.m, op.m, sizeof(to.m));
        }
        for (int j = 0; j < kLaneQubits; ++j)
            if (cur_lane[j] != lt[j]) throw DeviceError("internal: a lane exchange was not undone within its phase");
        Q.op_end = static_cast<uint16_t>(ko);
    }
    // Bits every op needs at 1 outside the tile: local ones shrink the tile
    // enumeration (the other tiles are left untouched in HBM: a lone
    // controlled gate reads and writes half the state), rank ones skip the
    // shard (the reference's rank-id control skip, distributed.cpp:143-145)
    uint64_t common = ~uint64_t{0};
    for (int k = 0; k < P.phases[P.num_phases - 1].op_end; ++k)
        if ((P.ops[k].hdr & 63) != TC_LANE_XCHG) common &= P.ops[k].outer_cmask; // (exchanges: pure moves)
    const uint64_t local_mask = local_len - 1;
    P.skip_ones = common & local_mask;
    const uint64_t rank_need = common & ~local_mask;
    P.num_tiles >>= __builtin_popcountll(P.skip_ones);
    if (plan_sink) { // (dry run with QGPU_PLAN_JIT_DUMP)
        jit_dump_program(P, std::getenv("QGPU_PLAN_JIT_DUMP"), static_cast<int>(passes));
        ++passes;
        return;
    }
    if (pass_stats_enabled()) record_pass_stats(P);
    ProfScope prof(env, PK_PASS, pass_profile_info(P));
    for (auto& s : shards) {
        P.global_offset = goff(s);
        if ((P.global_offset & rank_need) != rank_need) continue;
        launch_tile_pass(s.amps, P, env->stream);
    }
    cuda_check(cudaGetLastError(), "tile pass launch");
    ++passes;
}

void QuregImpl::launch_fused() {
    const int H = pass_H();
    std::vector<int> r = regs;
    for (int q = local_qubits - 1; static_cast<int>(r.size()) < H && q >= kLaneQubits; --q)
        if (std::find(r.begin(), r.end(), q) == r.end()) r.push_back(q);
    std::sort(r.begin(), r.end());

    PassParams P;
    std::memset(&P, 0, sizeof(P));
    P.num_tiles = uint64_t{1} << (local_qubits - kLaneQubits - H);
    P.H = H;
    P.num_ops = static_cast<int>(pending.size());
    uint64_t reg_bits = 0;
    for (int j = 0; j < H; ++j) {
        P.reg_pos[j] = r[j];
        reg_bits |= uint64_t{1} << r[j];
    }
    for (int i = 0; i < (1 << H); ++i) {
        uint64_t off = 0;
        for (int j = 0; j < H; ++j)
            if ((i >> j) & 1) off |= uint64_t{1} << r[j];
        P.reg_off[i] = off;
    }
    auto loc = [&](int q) -> QubitLoc {
        if (q < 0) return QubitLoc{LOC_OUTER, 0};
        if (q < kLaneQubits) return QubitLoc{LOC_LANE, static_cast<uint8_t>(q)};
        for (int j = 0; j < H; ++j)
            if (r[j] == q) return QubitLoc{LOC_REG, static_cast<uint8_t>(j)};
        return QubitLoc{LOC_OUTER, static_cast<uint8_t>(q)};
    };
    for (size_t k = 0; k < pending.size(); ++k) {
        const FlatOp& op = pending[k];
        PassOp& po = P.ops[k];
        switch (op.kind) {
        case FK_GATE:
            po.kind = op.cls == CLS_DIAG ? PO_DIAG
                                         : (op.q0 < kLaneQubits ? PO_PAIR_LANE : PO_PAIR_REG);
            break;
        case FK_DEPHASE: po.kind = PO_DEPHASE; break;
        default: po.kind = PO_COLLAPSE; break;
        }
        po.cls = op.cls;
        po.flags = op.kind == FK_COLLAPSE ? (op.q1 >= 0 ? 1 : 0) : op.flags;
        po.outcome = op.outcome;
        po.q0 = loc(op.q0);
        po.q1 = loc(op.q1);
        po.lane_cmask = static_cast<uint32_t>(op.cmask & ((1u << kLaneQubits) - 1));
        po.reg_cmask = 0;
        for (int j = 0; j < H; ++j)
            if ((op.cmask >> r[j]) & 1) po.reg_cmask |= 1u << j;
        po.outer_cmask = op.cmask & ~uint64_t{(1u << kLaneQubits) - 1} & ~reg_bits;
        std::memcpy(po.m, op.m, sizeof(po.m));
    }
    ProfScope prof(env, PK_PASS);
    for (auto& s : shards) {
        P.global_offset = goff(s);
        launch_pass(static_cast<double2*>(s.amps), P, env->stream); // double only (see enqueue_phys)
    }
    cuda_check(cudaGetLastError(), "fused pass launch");
    ++passes;
}

void QuregImpl::run_simple(const FlatOp& op) {
    ProfScope prof(env, PK_SIMPLE);
    for (auto& s : shards) {
        switch (op.kind) {
        case FK_GATE:
            if (op.cls == CLS_DIAG) {
                Mat2 m;
                std::memcpy(m.m, op.m, sizeof(m.m));
                launch_diag_simple(s.amps, single, local_len, goff(s), op.q0, op.cmask, m, op.flags,
                                   env->stream);
            } else {
                const uint64_t rank_mask = op.cmask >> local_qubits;
                if ((static_cast<uint64_t>(s.rank) & rank_mask) != rank_mask) break;
                Mat2 m;
                std::memcpy(m.m, op.m, sizeof(m.m));
                launch_gate_simple(s.amps, single, local_qubits, op.q0, op.cmask & (local_len - 1), m,
                                   op.cls, env->stream);
            }
            break;
        case FK_DEPHASE:
            launch_dephase(s.amps, single, local_len, goff(s), op.q0, op.q1, op.m[0], env->stream);
            break;
        case FK_COLLAPSE:
            launch_collapse(s.amps, single, local_len, goff(s), op.q0, op.q1, op.outcome, op.m[0],
                            env->stream);
            break;
        default: break;
        }
    }
    cuda_check(cudaGetLastError(), "kernel launch");
}

// ---------------------------------------------------------------- exchange

namespace {

struct ExchangeEvents {
    cudaEvent_t start = nullptr, recv[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
    explicit ExchangeEvents() {
        cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
        for (int i = 0; i < 2; ++i) {
            cudaEventCreateWithFlags(&recv[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
        }
    }
    ~ExchangeEvents() {
        cudaEventDestroy(start);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(recv[i]);
            cudaEventDestroy(done[i]);
        }
    }
};

} // namespace

// Pairwise sub-chunked exchange + combine. `combine(shard, chunk_ptr,
// recv_ptr, len, idx0)` writes only the shard's own half
// (distributed.cpp:174-187); chunk j is sent before combine(j) overwrites it
// (the in-place ordering rule of the PerAmplitude strategy, :215-231).
template <class Combine>
static void exchange_rounds(QuregImpl& q, int rank_bit, uint64_t rank_mask, uint64_t chunk,
                            Combine&& combine) {
    Env* env = q.env;
    const uint64_t bytes = chunk * q.amp_bytes();
    if (env->mode == Mode::Nccl) {
        Shard& s = q.shards[0];
        if ((static_cast<uint64_t>(s.rank) & rank_mask) != rank_mask) return;
        const int peer = s.rank ^ (1 << rank_bit);
        ExchangeEvents ev;
        cuda_check(cudaEventRecord(ev.start, env->stream), "event");
        cuda_check(cudaStreamWaitEvent(env->comm_stream, ev.start, 0), "event");
        uint64_t j = 0;
        for (uint64_t c0 = 0; c0 < q.local_len; c0 += chunk, ++j) {
            const int b = static_cast<int>(j & 1);
            if (j >= 2) cuda_check(cudaStreamWaitEvent(env->comm_stream, ev.done[b], 0), "event");
            env->nccl->sendrecv(peer, q.at(s.amps, c0), q.recv[b], bytes, env->comm_stream);
            cuda_check(cudaEventRecord(ev.recv[b], env->comm_stream), "event");
            cuda_check(cudaStreamWaitEvent(env->stream, ev.recv[b], 0), "event");
            combine(s, q.at(s.amps, c0), q.recv[b], chunk, c0);
            cuda_check(cudaEventRecord(ev.done[b], env->stream), "event");
            s.messages += 1;
            s.bytes += bytes;
        }
        // events are destroyed after the stream consumed them (the runtime
        // defers destruction of recorded events).
        return;
    }
    // Loopback: 2^k virtual ranks on this device; each pair's cell copies both
    // directions (InProcessTransport::exchange, transport.cpp:39-50).
    for (auto& s : q.shards) {
        const int peer = s.rank ^ (1 << rank_bit);
        if (peer < s.rank) continue;
        if ((static_cast<uint64_t>(s.rank) & rank_mask) != rank_mask) continue;
        Shard& p = q.shards[peer];
        for (uint64_t c0 = 0; c0 < q.local_len; c0 += chunk) {
            cuda_check(memcpy_counted(q.recv[0], q.at(p.amps, c0), bytes, cudaMemcpyDeviceToDevice,
                                       env->stream),
                       "loopback exchange");
            cuda_check(memcpy_counted(q.recv[1], q.at(s.amps, c0), bytes, cudaMemcpyDeviceToDevice,
                                       env->stream),
                       "loopback exchange");
            combine(s, q.at(s.amps, c0), q.recv[0], chunk, c0);
            combine(p, q.at(p.amps, c0), q.recv[1], chunk, c0);
            s.messages += 1;
            s.bytes += bytes;
            p.messages += 1;
            p.bytes += bytes;
        }
    }
}

void QuregImpl::run_exchange_gate(const FlatOp& op) {
    const int rank_bit = op.q0 - local_qubits;
    const uint64_t rank_mask = op.cmask >> local_qubits;
    const uint64_t low_mask = op.cmask & (local_len - 1);
    const uint64_t chunk = std::min<uint64_t>(env->chunk_amps, local_len);
    Mat2 m;
    std::memcpy(m.m, op.m, sizeof(m.m));
    if (env->mode == Mode::Peer) {
        // fused exchange + combine over peer memory: the pair (own_lo rank's
        // element i, partner's element i) is updated by one GPU, each rank
        // taking half of the local indices; no staging buffer
        Shard& s = shards[0];
        const bool active = (static_cast<uint64_t>(s.rank) & rank_mask) == rank_mask; // :141-145
        const int peer = s.rank ^ (1 << rank_bit);
        const std::vector<int> wait = active ? std::vector<int>{peer} : std::vector<int>{};
        env->peer->fence(env->stream, wait); // both partitions quiescent
        if (active) {
            ProfScope prof(env, PK_EXCHANGE);
            const int own_lo = ((s.rank >> rank_bit) & 1) == 0;
            void* lo_side = own_lo ? s.amps : peer_amps[peer];
            void* hi_side = own_lo ? peer_amps[peer] : s.amps;
            const uint64_t half = local_len / 2;
            launch_peer_combine(lo_side, hi_side, single, own_lo ? 0 : half, own_lo ? half : local_len - half,
                                low_mask, m, op.cls, env->stream);
            cuda_check(cudaGetLastError(), "peer exchange combine");
            s.messages += 1;
            s.bytes += local_len * amp_bytes();
        }
        env->peer->fence(env->stream, wait); // the partner's writes into this partition landed
        ++passes;
        return;
    }
    ensure_recv(chunk);
    ProfScope prof(env, PK_EXCHANGE);
    exchange_rounds(*this, rank_bit, rank_mask, chunk,
                    [&](Shard& s, void* mine, void* theirs, uint64_t len, uint64_t idx0) {
                        const int own_lo = ((s.rank >> rank_bit) & 1) == 0;
                        launch_combine(mine, theirs, single, len, idx0, low_mask, own_lo, m, op.cls,
                                       env->stream);
                    });
    cuda_check(cudaGetLastError(), "exchange combine");
    ++passes;
}

void QuregImpl::run_depol(const FlatOp& op) {
    const double keep = op.m[0], swap = op.m[1], off = op.m[2];
    ProfScope prof(env, PK_DEPOL);
    if (op.q1 < local_qubits) {
        for (auto& s : shards)
            launch_depolarise(s.amps, single, local_qubits, op.q0, op.q1, keep, swap, off, env->stream);
        cuda_check(cudaGetLastError(), "depolarise");
        ++passes;
        return;
    }
    const int rank_bit = op.q1 - local_qubits;
    if (env->mode == Mode::Peer) {
        // corner pairs (col-0 rank's element i, col-1 rank's element i | 2^t)
        // split between the two ranks; each scales its own off-diagonal half
        Shard& s = shards[0];
        const int own_col = (s.rank >> rank_bit) & 1;
        const int peer = s.rank ^ (1 << rank_bit);
        env->peer->fence(env->stream, {peer});
        void* col0 = own_col == 0 ? s.amps : peer_amps[peer];
        void* col1 = own_col == 0 ? peer_amps[peer] : s.amps;
        const uint64_t pairs = local_len / 2;
        launch_peer_combine_depol(col0, col1, single, own_col ? pairs / 2 : 0,
                                  own_col ? pairs - pairs / 2 : pairs / 2, op.q0, keep, swap, env->stream);
        launch_scale_bit(s.amps, single, local_len, op.q0, own_col ^ 1, off, env->stream);
        cuda_check(cudaGetLastError(), "peer depolarise");
        s.messages += 1;
        s.bytes += pairs * amp_bytes();
        env->peer->fence(env->stream, {peer});
        ++passes;
        return;
    }
    uint64_t chunk = std::min<uint64_t>(env->chunk_amps, local_len);
    chunk = std::max<uint64_t>(chunk, uint64_t{2} << op.q0);
    ensure_recv(chunk);
    exchange_rounds(*this, rank_bit, 0, chunk,
                    [&](Shard& s, void* mine, void* theirs, uint64_t len, uint64_t idx0) {
                        const int own_col = (s.rank >> rank_bit) & 1;
                        launch_combine_depol(mine, theirs, single, len, idx0, op.q0, own_col, keep, swap,
                                             off, env->stream);
                    });
    cuda_check(cudaGetLastError(), "depolarise exchange");
    ++passes;
}

// ------------------------------------------------------------ qubit swaps

// Trade physical global position g (rank bit j = g - local) with local
// position v: rank r (bit j = a) keeps the amplitudes whose local bit v is a
// and trades the half with bit v = !a with partner r ^ 2^j; both sides send
// and receive the same local offsets (a pure copy, in sub-chunks of
// min(chunk, 2^v) contiguous amplitudes, double-buffered like the exchange
// gates).
void QuregImpl::run_swap(int g, int v, bool flush) {
    // queued ops (e.g. restore_identity's local swaps) run first; the
    // light-cone drain has already run the ones on the traded positions
    if (flush) {
        flush_pass();
    } else if (!pending.empty()) { // (the open pass; the window stays)
        launch_tile();
        discard();
    }
    if (swap_sink) { // dry run (qgpuPlanDistributed)
        swap_sink->push_back({g, v});
        return;
    }
    const int j = g - local_qubits;
    const uint64_t block = uint64_t{1} << v;
    const uint64_t unit = std::min<uint64_t>(std::min<uint64_t>(env->chunk_amps, block), local_len / 2);
    const uint64_t units = (local_len / 2) / unit;
    ensure_recv(unit);
    const uint64_t bytes = unit * amp_bytes();
    // offset of the u-th unit of the half whose bit v == side
    auto offset = [&](uint64_t u, int side) {
        const uint64_t e = u * unit;                      // element index within the half
        const uint64_t hi = e >> v, lo = e & (block - 1); // deposit a zero... then set bit v
        return (hi << (v + 1)) | (static_cast<uint64_t>(side) << v) | lo;
    };
    ProfScope prof(env, PK_SWAP);
    if (env->mode == Mode::Peer) {
        // one kernel per rank moves half of the traded pairs both ways over
        // peer memory (in place, no staging buffer)
        Shard& s = shards[0];
        const int a = (s.rank >> j) & 1;
        const int peer = s.rank ^ (1 << j);
        env->peer->fence(env->stream, {peer});
        const uint64_t half = local_len / 2;
        launch_peer_swap(s.amps, peer_amps[peer], single, a ? half / 2 : 0, a ? half - half / 2 : half / 2, v,
                         a ^ 1, env->stream);
        cuda_check(cudaGetLastError(), "peer swap");
        s.messages += 1;
        s.bytes += half * amp_bytes();
        env->peer->fence(env->stream, {peer});
        ++passes;
        return;
    }
    if (env->mode == Mode::Nccl) {
        Shard& s = shards[0];
        const int a = (s.rank >> j) & 1;
        const int peer = s.rank ^ (1 << j);
        ExchangeEvents ev;
        cuda_check(cudaEventRecord(ev.start, env->stream), "event");
        cuda_check(cudaStreamWaitEvent(env->comm_stream, ev.start, 0), "event");
        for (uint64_t u = 0; u < units; ++u) {
            const int b = static_cast<int>(u & 1);
            void* mine = at(s.amps, offset(u, a ^ 1));
            if (u >= 2) cuda_check(cudaStreamWaitEvent(env->comm_stream, ev.done[b], 0), "event");
            env->nccl->sendrecv(peer, mine, recv[b], bytes, env->comm_stream);
            cuda_check(cudaEventRecord(ev.recv[b], env->comm_stream), "event");
            cuda_check(cudaStreamWaitEvent(env->stream, ev.recv[b], 0), "event");
            cuda_check(memcpy_counted(mine, recv[b], bytes, cudaMemcpyDeviceToDevice, env->stream),
                       "swap");
            cuda_check(cudaEventRecord(ev.done[b], env->stream), "event");
            s.messages += 1;
            s.bytes += bytes;
        }
    } else {
        for (auto& s : shards) {
            const int peer = s.rank ^ (1 << j);
            if (peer < s.rank) continue;
            Shard& p = shards[peer];
            // s has bit j = 0 (trades its bit-v = 1 half), p has bit j = 1
            for (uint64_t u = 0; u < units; ++u) {
                void* x = at(s.amps, offset(u, 1));
                void* y = at(p.amps, offset(u, 0));
                cuda_check(memcpy_counted(recv[0], x, bytes, cudaMemcpyDeviceToDevice, env->stream), "swap");
                cuda_check(memcpy_counted(x, y, bytes, cudaMemcpyDeviceToDevice, env->stream), "swap");
                cuda_check(memcpy_counted(y, recv[0], bytes, cudaMemcpyDeviceToDevice, env->stream), "swap");
                s.messages += 1;
                s.bytes += bytes;
                p.messages += 1;
                p.bytes += bytes;
            }
        }
    }
    ++passes;
}

// Swap two local qubits with three CNOTs (pure amplitude moves: exact).
void QuregImpl::local_swap(int a, int b) {
    FlatOp x;
    x.kind = FK_GATE;
    x.m[2] = 1.0;
    x.m[4] = 1.0;
    x.cls = classify(x.m, &x.flags);
    for (int k = 0; k < 3; ++k) {
        x.q0 = k == 1 ? a : b;
        x.cmask = uint64_t{1} << (k == 1 ? b : a);
        enqueue_phys(x);
    }
}

void QuregImpl::restore_identity() {
    if (!swaps_on()) return;
    flush(); // drain the logical queue first: it may swap
    if (sp.identity()) return;
    for (int L = 0; L < flat; ++L) {
        const int P = sp.l2p[L], Q = L; // current and home position
        if (P == Q) continue;
        const bool pg = P >= local_qubits, qg = Q >= local_qubits;
        if (!pg && !qg) {
            local_swap(P, Q);
        } else if (pg != qg) {
            run_swap(pg ? P : Q, pg ? Q : P);
        } else { // both global: (P w)(Q w)(P w) = (P Q) through a local w
            const int w = sp.victim(0);
            run_swap(P, w);
            sp.apply(P, w);
            run_swap(Q, w);
            sp.apply(Q, w);
            run_swap(P, w);
            sp.apply(P, w);
            continue;
        }
        sp.apply(P, Q);
    }
    flush_pass();
}

// -------------------------------------------------------------- reductions

namespace {
struct HostDD {
    double hi = 0.0, lo = 0.0;
    void add(double xh, double xl) {
        const double s = hi + xh;
        const double bb = s - hi;
        const double e = (hi - (s - bb)) + (xh - bb);
        const double t = e + lo + xl;
        hi = s + t;
        lo = t - (hi - s);
    }
};
} // namespace

double QuregImpl::combine_results(int n) {
    std::vector<double2> host(std::max(n, env->num_ranks));
    if (env->mode == Mode::Peer && env->num_ranks > 1) {
        double2 mine;
        cuda_check(memcpy_counted(&mine, results, sizeof(double2), cudaMemcpyDeviceToHost, env->stream),
                   "reduction readback");
        cuda_check(cudaStreamSynchronize(env->stream), "reduction");
        env->peer->allgather(&mine, host.data(), sizeof(double2));
        n = env->num_ranks;
        HostDD acc;
        for (int i = 0; i < n; ++i) acc.add(host[i].x, host[i].y); // rank order
        return acc.hi + acc.lo;
    }
    if (env->mode == Mode::Nccl && env->num_ranks > 1) {
        env->nccl->allgather(results, results + 1, sizeof(double2), env->stream);
        cuda_check(memcpy_counted(host.data(), results + 1, env->num_ranks * sizeof(double2),
                                   cudaMemcpyDeviceToHost, env->stream),
                   "reduction readback");
        n = env->num_ranks;
        env->wait_stream(env->stream);
    } else {
        cuda_check(memcpy_counted(host.data(), results, n * sizeof(double2),
                                   cudaMemcpyDeviceToHost, env->stream),
                   "reduction readback");
    }
    cuda_check(cudaStreamSynchronize(env->stream), "reduction");
    HostDD acc;
    for (int i = 0; i < n; ++i) acc.add(host[i].x, host[i].y); // rank order
    return acc.hi + acc.lo;
}

double QuregImpl::reduce_sel_phys(uint64_t mask, uint64_t val) {
    ProfScope prof(env, PK_REDUCE);
    const uint64_t lmask = mask & (local_len - 1);
    const uint64_t rmask = mask >> local_qubits, rval = val >> local_qubits;
    for (size_t k = 0; k < shards.size(); ++k) {
        if ((static_cast<uint64_t>(shards[k].rank) & rmask) != rval) {
            cuda_check(cudaMemsetAsync(results + k, 0, sizeof(double2), env->stream), "reduce");
            continue;
        }
        launch_reduce_norm_sel(shards[k].amps, single, local_len, lmask, val & lmask, partials, results + k,
                               env->stream);
    }
    cuda_check(cudaGetLastError(), "reduce");
    return combine_results(static_cast<int>(shards.size()));
}

bool QuregImpl::marginals_usable() const {
    static const bool off = [] {
        const char* v = std::getenv("QGPU_MARGINALS");
        return v && std::string(v) == "0";
    }();
    return !off && !density && local_qubits >= kMarginalsMinQubits && flat <= 63;
}

void QuregImpl::compute_marginals() {
    flush();
    if (marg_version == version) return;
    const int m = local_qubits;
    const size_t per = static_cast<size_t>(1 + m);
    if (!marg_scratch) {
        const size_t nvec = std::max(shards.size(), static_cast<size_t>(env->num_ranks)) + 1;
        if (cudaMalloc(&marg_scratch, marginals_scratch_bytes(m)) != cudaSuccess ||
            cudaMalloc(&marg_dev, nvec * per * sizeof(double2)) != cudaSuccess) {
            cudaGetLastError();
            throw ResourceError("failed to allocate the marginals scratch");
        }
    }
    {
        ProfScope prof(env, PK_REDUCE);
        for (size_t k = 0; k < shards.size(); ++k)
            launch_marginals(shards[k].amps, single, m, marg_scratch, marg_dev + k * per, env->stream);
        cuda_check(cudaGetLastError(), "marginals");
    }
    // every rank's vector on every rank, merged in rank order
    const int nr = env->num_ranks;
    std::vector<double2> all(static_cast<size_t>(nr) * per);
    if (!env->multi_process() || env->num_ranks == 1) { // every shard in this process
        cuda_check(memcpy_counted(all.data(), marg_dev, all.size() * sizeof(double2), cudaMemcpyDeviceToHost,
                                  env->stream),
                   "marginals");
        cuda_check(cudaStreamSynchronize(env->stream), "marginals");
    } else if (env->mode == Mode::Peer) {
        std::vector<double2> mine(per);
        cuda_check(memcpy_counted(mine.data(), marg_dev, per * sizeof(double2), cudaMemcpyDeviceToHost, env->stream),
                   "marginals");
        cuda_check(cudaStreamSynchronize(env->stream), "marginals");
        env->peer->allgather(mine.data(), all.data(), per * sizeof(double2));
    } else {
        env->nccl->allgather(marg_dev, marg_dev + per, per * sizeof(double2), env->stream);
        cuda_check(memcpy_counted(all.data(), marg_dev + per, all.size() * sizeof(double2), cudaMemcpyDeviceToHost,
                                  env->stream),
                   "marginals");
        env->wait_stream(env->stream);
    }
    struct Acc {
        double hi = 0.0, lo = 0.0;
        void add(double2 v) {
            const double s = hi + v.x, bb = s - hi;
            const double e = (hi - (s - bb)) + (v.x - bb);
            const double t = e + lo + v.y;
            hi = s + t;
            lo = t - (hi - s);
        }
    };
    std::vector<Acc> phys(static_cast<size_t>(flat) + 1);
    for (int r = 0; r < nr; ++r) { // rank order
        const double2* v = all.data() + static_cast<size_t>(r) * per;
        phys[0].add(v[0]);
        for (int q = 0; q < m; ++q) phys[1 + q].add(v[1 + q]);
        for (int g = m; g < flat; ++g)
            if ((r >> (g - m)) & 1) phys[1 + g].add(v[0]);
    }
    marg.assign(static_cast<size_t>(flat) + 1, make_double2(0.0, 0.0));
    marg[0] = make_double2(phys[0].hi, phys[0].lo);
    for (int L = 0; L < flat; ++L) {
        const int P = swaps_on() ? sp.l2p[L] : L;
        marg[1 + L] = make_double2(phys[1 + P].hi, phys[1 + P].lo);
    }
    marg_version = version;
}

double QuregImpl::reduce_norm(int t, int outcome) {
    if (!density && !deferred.empty() && lq.empty() && pending.empty()) {
        // pending collapses as a selection (logical qubits), scaled by their
        // scale^2; the state in HBM is the pre-collapse one
        uint64_t m = 0, v = 0;
        double s2 = 1.0;
        bool empty = false;
        for (const FlatOp& op : deferred) {
            const uint64_t b = uint64_t{1} << op.q0;
            if ((m & b) && (((v >> op.q0) & 1u) != op.outcome)) empty = true;
            m |= b;
            v |= static_cast<uint64_t>(op.outcome) << op.q0;
            s2 *= op.m[0] * op.m[0];
        }
        if (t >= 0) {
            const uint64_t b = uint64_t{1} << t;
            if ((m & b) && (((v >> t) & 1u) != static_cast<uint64_t>(outcome))) empty = true;
            m |= b;
            v |= static_cast<uint64_t>(outcome) << t;
        }
        const uint64_t pm = swaps_on() ? sp.phys_mask(m) : m, pv = swaps_on() ? sp.phys_mask(v) : v;
        if (__builtin_popcountll(pm & (local_len - 1)) <= 8) {
            const double r = reduce_sel_phys(pm, pv); // collective: every rank reduces
            return empty ? 0.0 : r * s2;
        }
    }
    if (t >= 0 && marginals_usable()) {
        compute_marginals();
        const double2 p1 = marg[1 + t];
        if (outcome) return p1.x + p1.y;
        // total - P(1) in double-double, then rounded
        const double2 tot = marg[0];
        const double s = tot.x - p1.x, bb = s - tot.x;
        const double e = (tot.x - (s - bb)) + (-p1.x - bb);
        return s + (e + tot.y - p1.y);
    }
    flush();
    if (swaps_on()) t = sp.phys(t);
    ProfScope prof(env, PK_REDUCE);
    for (size_t k = 0; k < shards.size(); ++k)
        launch_reduce_norm(shards[k].amps, single, local_len, goff(shards[k]), t, outcome, partials,
                           results + k, env->stream);
    cuda_check(cudaGetLastError(), "reduce");
    return combine_results(static_cast<int>(shards.size()));
}

double QuregImpl::reduce_diag(int t, int outcome, int comp) {
    restore_identity(); // the diagonal is j == k in the logical layout
    flush();
    ProfScope prof(env, PK_REDUCE);
    for (size_t k = 0; k < shards.size(); ++k)
        launch_reduce_diag(shards[k].amps, single, local_len, goff(shards[k]), N, t, outcome, comp,
                           partials, results + k, env->stream);
    cuda_check(cudaGetLastError(), "reduce");
    return combine_results(static_cast<int>(shards.size()));
}

Complex QuregImpl::trace() {
    // density.cpp:147-154 sums both parts of the diagonal.
    Complex c;
    c.real = reduce_diag(-1, 0, 0);
    c.imag = reduce_diag(-1, 0, 1);
    return c;
}

void QuregImpl::get_raw(uint64_t start, uint64_t num, void* out) {
    restore_identity();
    flush();
    const uint64_t end = start + num;
    if (env->mode == Mode::Peer && env->num_ranks > 1 && num == 1) {
        // single amplitude: the owner contributes it through the mailboxes
        const uint64_t lo = goff(shards[0]);
        const int owner = static_cast<int>(start >> local_qubits);
        double2 mine = make_double2(0.0, 0.0);
        if (owner == shards[0].rank) {
            cuda_check(memcpy_counted(&mine, at(shards[0].amps, start - lo), amp_bytes(), cudaMemcpyDeviceToHost,
                                       env->stream),
                       "read");
            cuda_check(cudaStreamSynchronize(env->stream), "read");
        }
        std::vector<double2> all(env->num_ranks);
        env->peer->allgather(&mine, all.data(), sizeof(double2));
        std::memcpy(out, &all[owner], amp_bytes());
        return;
    }
    if (env->multi_process() && env->num_ranks > 1) {
        if (num != 1) {
            const uint64_t lo = goff(shards[0]), hi = lo + local_len;
            if (start < lo || end > hi)
                throw DomainError("bulk reads are limited to this rank's amplitudes [" +
                                  std::to_string(lo) + ", " + std::to_string(hi) + ")");
            cuda_check(memcpy_counted(out, at(shards[0].amps, start - lo), num * amp_bytes(),
                                       cudaMemcpyDeviceToHost, env->stream),
                       "read");
            cuda_check(cudaStreamSynchronize(env->stream), "read");
            return;
        }
        // single amplitude: the owner contributes it, everyone gets it.
        const uint64_t lo = goff(shards[0]);
        const int owner = static_cast<int>(start >> local_qubits);
        double2 zero = make_double2(0.0, 0.0);
        if (owner == shards[0].rank)
            cuda_check(memcpy_counted(results, at(shards[0].amps, start - lo), amp_bytes(),
                                       cudaMemcpyDeviceToDevice, env->stream),
                       "read");
        else
            cuda_check(memcpy_counted(results, &zero, sizeof(double2), cudaMemcpyHostToDevice,
                                       env->stream),
                       "read");
        env->nccl->allgather(results, results + 1, sizeof(double2), env->stream);
        cuda_check(memcpy_counted(out, results + 1 + owner, amp_bytes(),
                                   cudaMemcpyDeviceToHost, env->stream),
                   "read");
        cuda_check(cudaStreamSynchronize(env->stream), "read");
        return;
    }
    for (auto& s : shards) {
        const uint64_t lo = goff(s), hi = lo + local_len;
        const uint64_t a = std::max(lo, start), b = std::min(hi, end);
        if (a >= b) continue;
        cuda_check(memcpy_counted(at(out, a - start), at(s.amps, a - lo), (b - a) * amp_bytes(),
                                   cudaMemcpyDeviceToHost, env->stream),
                   "read");
    }
    cuda_check(cudaStreamSynchronize(env->stream), "read");
}

void QuregImpl::set_raw(uint64_t start, uint64_t num, const void* in) {
    restore_identity();
    flush();
    ++version;
    const uint64_t end = start + num;
    for (auto& s : shards) {
        const uint64_t lo = goff(s), hi = lo + local_len;
        const uint64_t a = std::max(lo, start), b = std::min(hi, end);
        if (a >= b) continue;
        cuda_check(memcpy_counted(at(s.amps, a - lo), at(const_cast<void*>(in), a - start), (b - a) * amp_bytes(),
                                   cudaMemcpyHostToDevice, env->stream),
                   "write");
    }
    cuda_check(cudaStreamSynchronize(env->stream), "write");
}

// The host boundary is double in both precisions: single-precision registers
// widen on read and narrow on write (AmpVector::get / set, register.cpp:30-51).
void QuregImpl::get_flat(uint64_t start, uint64_t num, double2* out) {
    if (!single) {
        get_raw(start, num, out);
        return;
    }
    std::vector<float2> tmp(num);
    get_raw(start, num, tmp.data());
    for (uint64_t i = 0; i < num; ++i) out[i] = make_double2(tmp[i].x, tmp[i].y);
}

void QuregImpl::set_flat(uint64_t start, uint64_t num, const double2* in) {
    if (!single) {
        set_raw(start, num, in);
        return;
    }
    std::vector<float2> tmp(num);
    for (uint64_t i = 0; i < num; ++i)
        tmp[i] = make_float2(static_cast<float>(in[i].x), static_cast<float>(in[i].y));
    set_raw(start, num, tmp.data());
}

} // namespace qgpu
