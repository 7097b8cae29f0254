// api.cpp — the extern "C" boundary (include/QuEST.h, include/qgpu.h).
//
// Every entry point validates its arguments on the host with the reference's
// rules BEFORE touching device state (the reference throws DomainError before
// mutation: kernels.cpp:22-41, density.cpp:17-22, 118-145,
// register.cpp:31-53, 101-117), then queues the operation on the register.
// Exceptions never cross the ABI: they are converted to the error handler
// (QuEST's invalidQuESTInputError) plus a thread-local code/message.
#include "QuEST.h"
#include "qgpu.h"

#include "qgpu_kernels.h"
#include "runtime.h"
#include "peer.h"
#include "transport.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <mutex>
#include <numbers>
#include <string>
#include <unistd.h>
#include <unordered_set>
#include <vector>

using namespace qgpu;

// ------------------------------------------------------------------ errors

namespace {

thread_local int t_code = QGPU_OK;
thread_local std::string t_msg;
qgpuErrorHandler g_handler = nullptr;
void* g_handler_user = nullptr;

std::mutex g_live_mu;
std::unordered_set<QuregImpl*> g_live; // handle validation
std::unordered_set<Env*> g_envs;

void report(int code, const std::string& msg, const char* func) {
    t_code = code;
    t_msg = msg;
    if (g_handler)
        g_handler(t_msg.c_str(), func, code, g_handler_user);
    else
        invalidQuESTInputError(t_msg.c_str(), func);
}

// A transport or device failure inside a collective leaves the partner
// ranks blocked; fail them fast instead: peer groups get the message
// (their barriers throw CommError), NCCL communicators are aborted.
void abort_groups(const std::string& msg) {
    std::lock_guard<std::mutex> lk(g_live_mu);
    for (Env* e : g_envs) {
        if (e->peer) e->peer->abort("rank " + std::to_string(e->rank) + ": " + msg);
        if (e->nccl) e->nccl->abort();
    }
}

template <class F, class R>
R guarded(const char* func, R fallback, F&& f) {
    t_code = QGPU_OK;
    t_msg.clear();
    try {
        return f();
    } catch (const qgpu::DomainError& e) {
        report(QGPU_DOMAIN_ERROR, e.what(), func);
    } catch (const qgpu::ResourceError& e) {
        report(QGPU_RESOURCE_ERROR, e.what(), func);
    } catch (const qgpu::CommError& e) {
        abort_groups(std::string(func) + ": " + e.what());
        report(QGPU_COMM_ERROR, e.what(), func);
    } catch (const qgpu::DeviceError& e) {
        abort_groups(std::string(func) + ": " + e.what());
        report(QGPU_DEVICE_ERROR, e.what(), func);
    } catch (const std::bad_alloc&) {
        report(QGPU_RESOURCE_ERROR, "host allocation failed", func);
    } catch (const std::exception& e) {
        report(QGPU_DEVICE_ERROR, e.what(), func);
    }
    return fallback;
}

template <class F>
void guarded_void(const char* func, F&& f) {
    guarded(func, 0, [&] {
        f();
        return 0;
    });
}

Env* env_of(QuESTEnv env) {
    Env* e = static_cast<Env*>(env.impl);
    std::lock_guard<std::mutex> lk(g_live_mu);
    if (!e || !g_envs.count(e)) throw qgpu::DomainError("invalid QuESTEnv handle");
    return e;
}

QuregImpl* reg_of(Qureg q) {
    QuregImpl* r = static_cast<QuregImpl*>(q.impl);
    std::lock_guard<std::mutex> lk(g_live_mu);
    if (!r || !g_live.count(r)) throw qgpu::DomainError("invalid or destroyed Qureg handle");
    return r;
}

// ------------------------------------------------------------- validation

// require_ket_qubit (density.cpp:17-22) / make_control_mask target check
// (kernels.cpp:24-28).
void check_qubit(const QuregImpl* r, int q, const char* role) {
    if (q < 0 || q >= r->N) {
        if (r->density)
            throw qgpu::DomainError("invalid qubit " + std::to_string(q) + " for " +
                                    std::to_string(r->N) + "-qubit density matrix");
        throw qgpu::DomainError(std::string("invalid ") + role + " qubit " + std::to_string(q) +
                                " for " + std::to_string(r->N) + "-qubit vector");
    }
}

// kernels.cpp:22-41 (on the represented qubits; density registers shift the
// mask to the bra half themselves).
uint64_t control_mask(const QuregImpl* r, const int* controls, int n, int target) {
    check_qubit(r, target, "target");
    uint64_t mask = 0;
    for (int i = 0; i < n; ++i) {
        const int c = controls[i];
        if (c < 0 || c >= r->N) {
            if (r->density)
                throw qgpu::DomainError("invalid qubit " + std::to_string(c) + " for " +
                                        std::to_string(r->N) + "-qubit density matrix");
            throw qgpu::DomainError("invalid control qubit " + std::to_string(c));
        }
        if (c == target)
            throw qgpu::DomainError("control qubit " + std::to_string(c) + " overlaps the target");
        const uint64_t bit = uint64_t{1} << c;
        if (mask & bit) throw qgpu::DomainError("duplicate control qubit " + std::to_string(c));
        mask |= bit;
    }
    return mask;
}

void require_density(const QuregImpl* r, const char* what) {
    if (!r->density)
        throw qgpu::DomainError(std::string(what) + " requires a density-matrix register");
}

void require_statevec(const QuregImpl* r, const char* what) {
    if (r->density)
        throw qgpu::DomainError(std::string(what) + " requires a state-vector register");
}

// ------------------------------------------------------- gate matrices (L2)

struct M2 {
    double m[8];
};

M2 mat(double ar, double ai, double br, double bi, double cr, double ci, double dr, double di) {
    return M2{{ar, ai, br, bi, cr, ci, dr, di}};
}

// gates.cpp:51-98, evaluated with the same expressions so the doubles match.
M2 m_hadamard() {
    const double s = 1.0 / std::sqrt(2.0);
    return mat(s, 0, s, 0, s, 0, -s, 0);
}
M2 m_x() { return mat(0, 0, 1, 0, 1, 0, 0, 0); }
M2 m_y() { return mat(0, 0, 0, -1, 0, 1, 0, 0); }
M2 m_z() { return mat(1, 0, 0, 0, 0, 0, -1, 0); }
M2 m_t() {
    using std::numbers::pi;
    return mat(1, 0, 0, 0, 0, 0, std::cos(pi / 4), std::sin(pi / 4));
}
M2 m_s() { return mat(1, 0, 0, 0, 0, 0, 0, 1); }
M2 m_phase(double angle) { return mat(1, 0, 0, 0, 0, 0, std::cos(angle), std::sin(angle)); }
// rotation_matrix (gates.cpp:85-98): cos(a/2) I - i sin(a/2) (n . sigma).
M2 m_rotation(double nx, double ny, double nz, double angle) {
    const double c = std::cos(angle / 2), s = std::sin(angle / 2);
    return mat(c, -s * nz, -s * ny, -s * nx, s * ny, -s * nx, c, s * nz);
}
// QuEST normalises the axis; a unit axis (|n|^2 = 1 within 1e-12, the
// reference's acceptance, gates.cpp:87-90) is used exactly as given.
M2 m_axis(double angle, Vector axis) {
    const double len2 = axis.x * axis.x + axis.y * axis.y + axis.z * axis.z;
    if (!(len2 > 0.0) || !std::isfinite(len2))
        throw qgpu::DomainError("rotation axis must be a non-zero finite vector");
    if (std::abs(len2 - 1.0) > 1e-12) {
        const double n = std::sqrt(len2);
        axis.x /= n;
        axis.y /= n;
        axis.z /= n;
    }
    return m_rotation(axis.x, axis.y, axis.z, angle);
}
// compactUnitary: [[alpha, -conj(beta)], [beta, conj(alpha)]].
M2 m_compact(Complex a, Complex b) {
    const double norm = a.real * a.real + a.imag * a.imag + b.real * b.real + b.imag * b.imag;
    if (std::abs(norm - 1.0) > 1e-12)
        throw qgpu::DomainError("compact unitary requires |alpha|^2 + |beta|^2 = 1");
    return mat(a.real, a.imag, -b.real, b.imag, b.real, b.imag, a.real, -a.imag);
}

// is_unitary (gates.cpp:16-24): G^dagger G = I entrywise within tol.
bool is_unitary(const M2& g, double tol) {
    struct C {
        double r, i;
    };
    auto cj_mul = [](C a, C b) { return C{a.r * b.r + a.i * b.i, a.r * b.i - a.i * b.r}; };
    const C m00{g.m[0], g.m[1]}, m01{g.m[2], g.m[3]}, m10{g.m[4], g.m[5]}, m11{g.m[6], g.m[7]};
    auto add = [](C a, C b) { return C{a.r + b.r, a.i + b.i}; };
    const C e00 = add(cj_mul(m00, m00), cj_mul(m10, m10));
    const C e01 = add(cj_mul(m00, m01), cj_mul(m10, m11));
    const C e10 = add(cj_mul(m01, m00), cj_mul(m11, m10));
    const C e11 = add(cj_mul(m01, m01), cj_mul(m11, m11));
    auto mx = [](C a) { return std::max(std::abs(a.r), std::abs(a.i)); };
    return mx(C{e00.r - 1, e00.i}) <= tol && mx(e01) <= tol && mx(e10) <= tol &&
           mx(C{e11.r - 1, e11.i}) <= tol;
}

M2 from_cm2(const ComplexMatrix2& u) {
    return mat(u.real[0][0], u.imag[0][0], u.real[0][1], u.imag[0][1], u.real[1][0],
               u.imag[1][0], u.real[1][1], u.imag[1][1]);
}

M2 checked_unitary(const M2& g) {
    for (double x : g.m)
        if (!std::isfinite(x)) throw qgpu::DomainError("matrix entries must be finite");
    if (!is_unitary(g, 1e-12)) throw qgpu::DomainError("matrix is not unitary within tolerance");
    return g;
}

// Queues G on (target, controls): state vector -> one flat op
// (apply_controlled_gate, kernels.cpp:105-112); density matrix -> G at t and
// conj(G) at t+N with the controls shifted by N (density.cpp:85-116).
void apply_gate(QuregImpl* r, int target, uint64_t cmask, const M2& g) {
    FlatOp op;
    op.kind = FK_GATE;
    op.q0 = target;
    op.cmask = cmask;
    std::memcpy(op.m, g.m, sizeof(op.m));
    op.cls = classify(op.m, &op.flags);
    r->enqueue(op);
    if (r->density) {
        FlatOp b = op;
        b.q0 = target + r->N;
        b.cmask = cmask << r->N;
        for (int k = 1; k < 8; k += 2) b.m[k] = -op.m[k]; // GateMatrix::conjugate
        b.cls = classify(b.m, &b.flags);
        r->enqueue(b);
    }
}

void gate_call(const char* func, Qureg q, const int* controls, int nc, int target,
               const M2& g) {
    guarded_void(func, [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, controls, nc, target);
        apply_gate(r, target, mask, g);
    });
}

uint64_t splitmix_next(uint64_t* st) { // circuit.cpp:20-25
    uint64_t z = (*st += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t fold_seeds(const uint64_t* seeds, int n) {
    uint64_t st = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t tmp = st ^ seeds[i];
        st = splitmix_next(&tmp);
    }
    return st;
}

// Rank 0's value of `v` on every rank (one all-gather of 8 bytes).
uint64_t agree_on_rank0(Env* e, uint64_t v) {
    if (e->num_ranks <= 1) return v;
    std::vector<uint64_t> all(static_cast<size_t>(e->num_ranks));
    if (e->mode == Mode::Peer) {
        e->peer->allgather(&v, all.data(), sizeof(v));
        return all[0];
    }
    if (e->mode == Mode::Nccl) {
        uint64_t* d = nullptr;
        cuda_check(cudaMalloc(&d, sizeof(uint64_t) * (all.size() + 1)), "cudaMalloc");
        try {
            cuda_check(memcpy_counted(d, &v, sizeof(v), cudaMemcpyHostToDevice, e->stream), "seed");
            e->nccl->allgather(d, d + 1, sizeof(v), e->stream);
            cuda_check(memcpy_counted(all.data(), d + 1, sizeof(v) * all.size(), cudaMemcpyDeviceToHost,
                                       e->stream),
                       "seed");
            cuda_check(cudaStreamSynchronize(e->stream), "seed");
        } catch (...) {
            cudaFree(d);
            throw;
        }
        cudaFree(d);
        return all[0];
    }
    return v;
}

QuESTEnv make_env(Mode mode, int rank, int nranks, int device, const char* id128) {
    if (nranks < 1 || (nranks & (nranks - 1)))
        throw qgpu::DomainError("rank count must be a power of two, got " +
                                std::to_string(nranks));
    if (rank < 0 || rank >= nranks)
        throw qgpu::DomainError("invalid rank " + std::to_string(rank));
    auto e = std::make_unique<Env>();
    e->mode = mode;
    e->rank = rank;
    e->num_ranks = nranks;
    while ((1 << e->rank_log2) < nranks) ++e->rank_log2;
    if (device < 0) cuda_check(cudaGetDevice(&device), "cudaGetDevice");
    e->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&e->comm_stream, cudaStreamNonBlocking),
               "cudaStreamCreate");
    const uint64_t seeds[2] = {static_cast<uint64_t>(std::time(nullptr)),
                               static_cast<uint64_t>(getpid())};
    e->rng = fold_seeds(seeds, 2);
    if (const char* v = std::getenv("QGPU_TILE_TARGETS"))
        e->tile_targets = std::clamp(std::atoi(v), 1, qgpu::kTileHigh);
    if (const char* v = std::getenv("QGPU_ORDER")) {
        if (!std::strcmp(v, "exact") || !std::strcmp(v, "0")) e->order = 0;
        else if (!std::strcmp(v, "reorder") || !std::strcmp(v, "1")) e->order = 1;
        else throw qgpu::DomainError(std::string("QGPU_ORDER must be exact or reorder, got ") + v);
    }
    if (const char* v = std::getenv("QGPU_WINDOW")) e->window = std::clamp(std::atoi(v), 1, 65536);
    if (const char* v = std::getenv("QGPU_LANE_CAP")) e->lane_cap = std::max(0, std::atoi(v));
    if (const char* v = std::getenv("QGPU_NORMALIZE")) e->normalize = std::atoi(v); // (2: no symmetric lane diagonals)
    if (const char* v = std::getenv("QGPU_XCHG")) e->exchanges = std::atoi(v);
    if (const char* v = std::getenv("QGPU_MERGE")) e->merge = std::atoi(v) != 0;
    if (const char* v = std::getenv("QGPU_SWIZZLE")) e->swizzle = std::max(0, std::atoi(v));
    if (const char* v = std::getenv("QGPU_TILE_PHASES"))
        e->tile_phases = std::clamp(std::atoi(v), 1, qgpu::kMaxPhases);
    if (mode == Mode::Nccl && nranks > 1) e->nccl = std::make_unique<NcclComm>(rank, nranks, id128);
    if (mode == Mode::Peer) e->peer = std::make_unique<qgpu::PeerGroup>(rank, nranks, device, id128);
    // measure() draws its outcome from this state on every rank: all ranks
    // must hold rank 0's seed (QuEST broadcasts its default seed)
    e->rng = agree_on_rank0(e.get(), e->rng);
    QuESTEnv out;
    out.rank = mode == Mode::Loopback ? 0 : rank;
    out.numRanks = nranks;
    out.impl = e.get();
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_envs.insert(e.get());
    e.release();
    return out;
}

Qureg make_handle(QuregImpl* r) {
    Qureg q;
    q.isDensityMatrix = r->density ? 1 : 0;
    q.numQubitsRepresented = r->N;
    q.numQubitsInStateVec = r->flat;
    q.numAmpsPerChunk = static_cast<long long>(r->local_len);
    q.numAmpsTotal = static_cast<long long>(uint64_t{1} << r->flat);
    q.chunkId = r->env->multi_process() ? r->env->rank : 0;
    q.numChunks = r->env->num_ranks;
    q.impl = r;
    {
        std::lock_guard<std::mutex> lk(g_live_mu);
        g_live.insert(r);
    }
    return q;
}

Qureg null_qureg() {
    Qureg q;
    std::memset(&q, 0, sizeof(q));
    return q;
}

void check_index(const QuregImpl* r, long long idx) {
    const uint64_t len = uint64_t{1} << r->flat;
    if (idx < 0 || static_cast<uint64_t>(idx) >= len)
        throw qgpu::DomainError("amplitude index " + std::to_string(idx) + " out of range [0, " +
                                std::to_string(len) + ")");
}

double2 read_flat(QuregImpl* r, long long idx) {
    check_index(r, idx);
    double2 v;
    r->get_flat(static_cast<uint64_t>(idx), 1, &v);
    return v;
}

void check_outcome(int outcome) {
    if (outcome != 0 && outcome != 1)
        throw qgpu::DomainError("invalid measurement outcome " + std::to_string(outcome) +
                                " -- must be either 0 or 1");
}

double prob_of_outcome(QuregImpl* r, int t, int outcome) {
    return r->density ? r->reduce_diag(t, outcome) : r->reduce_norm(t, outcome);
}

void enqueue_collapse(QuregImpl* r, int t, int outcome, double prob) {
    FlatOp op;
    op.kind = FK_COLLAPSE;
    op.q0 = t;
    op.q1 = r->density ? t + r->N : -1;
    op.outcome = static_cast<uint8_t>(outcome);
    op.m[0] = r->density ? 1.0 / prob : 1.0 / std::sqrt(prob);
    if (r->density)
        r->enqueue(op);
    else
        r->defer_collapse(op); // fused into the next pass; reductions select around it
}

} // namespace

extern "C" {

// QuEST's override point. The library default only records (qgpuGetLastError);
// a program defining this symbol replaces it, as with QuEST.
__attribute__((weak)) void invalidQuESTInputError(const char* errMsg, const char* errFunc) {
    (void)errMsg;
    (void)errFunc;
}

void qgpuSetErrorHandler(qgpuErrorHandler handler, void* user) {
    g_handler = handler;
    g_handler_user = user;
}

int qgpuGetLastError(char* buf, int len) {
    if (buf && len > 0) {
        std::strncpy(buf, t_msg.c_str(), static_cast<size_t>(len - 1));
        buf[len - 1] = 0;
    }
    return t_code;
}

void qgpuClearError(void) {
    t_code = QGPU_OK;
    t_msg.clear();
}

const char* qgpuVersion(void) { return "qgpu 0.1 (sm_100a)"; }

unsigned long long qgpuKernelLaunches(void) { return qgpu::launch_count(); }

void qgpuTransferBytes(unsigned long long* h2d, unsigned long long* d2h) {
    uint64_t a = 0, b = 0;
    qgpu::transfer_bytes(&a, &b);
    if (h2d) *h2d = a;
    if (d2h) *d2h = b;
}

// ------------------------------------------------------------- environment

QuESTEnv createQuESTEnv(void) {
    QuESTEnv bad{0, 0, nullptr};
    return guarded("createQuESTEnv", bad, [] { return make_env(Mode::Single, 0, 1, -1, nullptr); });
}

QuESTEnv qgpuCreateLoopbackEnv(int numRanks) {
    QuESTEnv bad{0, 0, nullptr};
    return guarded("qgpuCreateLoopbackEnv", bad,
                   [&] { return make_env(Mode::Loopback, 0, numRanks, -1, nullptr); });
}

int qgpuGetNcclUniqueId(char* out128) {
    return guarded("qgpuGetNcclUniqueId", 1, [&] {
        NcclComm::unique_id(out128);
        return 0;
    });
}

QuESTEnv qgpuCreateNcclEnv(int rank, int numRanks, int device, const char* uniqueId128) {
    QuESTEnv bad{0, 0, nullptr};
    return guarded("qgpuCreateNcclEnv", bad,
                   [&] { return make_env(Mode::Nccl, rank, numRanks, device, uniqueId128); });
}

int qgpuPeerUniqueId(char* out128) {
    return guarded("qgpuPeerUniqueId", 1, [&] {
        if (!out128) throw qgpu::DomainError("null id buffer");
        qgpu::PeerGroup::unique_id(out128);
        return 0;
    });
}

QuESTEnv qgpuCreatePeerEnv(int rank, int numRanks, int device, const char* id128) {
    QuESTEnv bad{0, 0, nullptr};
    return guarded("qgpuCreatePeerEnv", bad, [&] {
        if (!id128) throw qgpu::DomainError("null peer group id");
        return make_env(Mode::Peer, rank, numRanks, device, id128);
    });
}

int qgpuPeerProbe(const char* id128, int rank, int numRanks, int rounds, int exitAfter) {
    return guarded("qgpuPeerProbe", static_cast<int>(QGPU_COMM_ERROR), [&] {
        if (!id128) throw qgpu::DomainError("null peer group id");
        qgpu::PeerGroup g(rank, numRanks, 0, id128, false);
        for (int it = 0; it < rounds; ++it) {
            if (it == exitAfter) std::_Exit(3); // a rank that dies mid-protocol
            const uint64_t mine = static_cast<uint64_t>(rank) * 1000003u + static_cast<uint64_t>(it);
            std::vector<uint64_t> all(static_cast<size_t>(numRanks));
            g.allgather(&mine, all.data(), sizeof(mine));
            for (int r = 0; r < numRanks; ++r)
                if (all[r] != static_cast<uint64_t>(r) * 1000003u + static_cast<uint64_t>(it))
                    throw qgpu::CommError("peer mailbox mismatch at round " + std::to_string(it));
            if (it % 7 == 0) g.barrier();
        }
        return 0;
    });
}

void destroyQuESTEnv(QuESTEnv env) {
    guarded_void("destroyQuESTEnv", [&] {
        Env* e = env_of(env);
        {
            std::lock_guard<std::mutex> lk(g_live_mu);
            for (QuregImpl* q : e->quregs) g_live.erase(q);
            g_envs.erase(e);
        }
        delete e;
    });
}

void syncQuESTEnv(QuESTEnv env) {
    guarded_void("syncQuESTEnv", [&] {
        Env* e = env_of(env);
        for (QuregImpl* q : e->quregs) q->flush();
        e->wait_stream(e->stream);
        cuda_check(cudaStreamSynchronize(e->comm_stream), "syncQuESTEnv");
        if (e->peer) e->peer->barrier(); // every rank's work finished (QuEST: MPI_Barrier)
    });
}

int syncQuESTSuccess(int successCode) { return successCode; }

void reportQuESTEnv(QuESTEnv env) {
    guarded_void("reportQuESTEnv", [&] {
        Env* e = env_of(env);
        cudaDeviceProp p;
        cuda_check(cudaGetDeviceProperties(&p, e->device), "cudaGetDeviceProperties");
        const char* mode = e->mode == Mode::Single     ? "single"
                           : e->mode == Mode::Loopback ? "loopback"
                           : e->mode == Mode::Peer     ? "peer"
                                                       : "nccl";
        std::printf("EXECUTION ENVIRONMENT:\nRunning on %s (sm_%d%d, %d SMs), %s mode, rank %d of %d\n",
                    p.name, p.major, p.minor, p.multiProcessorCount, mode, e->rank, e->num_ranks);
        std::printf("Fusion mode %d, max %d ops/pass, %d register qubits\nPrecision: complex double\n",
                    e->fusion_mode, e->max_ops, e->reg_qubits);
    });
}

void seedQuEST(QuESTEnv* env, unsigned long int* seedArray, int numSeeds) {
    guarded_void("seedQuEST", [&] {
        if (!env) throw qgpu::DomainError("null QuESTEnv");
        Env* e = env_of(*env);
        if (numSeeds < 0 || (numSeeds > 0 && !seedArray))
            throw qgpu::DomainError("invalid seed array");
        std::vector<uint64_t> s(seedArray, seedArray + numSeeds);
        e->rng = fold_seeds(s.data(), numSeeds);
    });
}

void seedQuESTDefault(QuESTEnv* env) {
    unsigned long int seeds[2] = {static_cast<unsigned long>(std::time(nullptr)),
                                  static_cast<unsigned long>(getpid())};
    seedQuEST(env, seeds, 2);
    guarded_void("seedQuESTDefault", [&] {
        if (!env) throw qgpu::DomainError("null QuESTEnv");
        Env* e = env_of(*env);
        e->rng = agree_on_rank0(e, e->rng); // rank 0's default seed everywhere
    });
}

void qgpuSetFusion(QuESTEnv env, int mode, int maxOps, int regQubits) {
    guarded_void("qgpuSetFusion", [&] {
        Env* e = env_of(env);
        if (mode < 0 || mode > 2) throw qgpu::DomainError("fusion mode must be 0, 1 or 2");
        if (maxOps > kMaxPassOps)
            throw qgpu::DomainError("at most " + std::to_string(kMaxPassOps) + " ops per pass");
        if (regQubits > kMaxRegQubits)
            throw qgpu::DomainError("at most " + std::to_string(kMaxRegQubits) +
                                    " register qubits");
        for (QuregImpl* q : e->quregs) q->flush();
        e->fusion_mode = mode;
        if (maxOps > 0) {
            e->max_ops = maxOps;
            e->tile_max_ops = maxOps;
        }
        if (regQubits > 0) e->reg_qubits = regQubits;
    });
}

void* qgpuGetStream(QuESTEnv env) {
    return guarded("qgpuGetStream", static_cast<void*>(nullptr),
                   [&] { return static_cast<void*>(env_of(env)->stream); });
}

int qgpuGetDevice(QuESTEnv env) {
    return guarded("qgpuGetDevice", -1, [&] { return env_of(env)->device; });
}

void qgpuSetExchangeChunk(QuESTEnv env, long long int amps) {
    guarded_void("qgpuSetExchangeChunk", [&] {
        Env* e = env_of(env);
        if (amps < 1 || (amps & (amps - 1)))
            throw qgpu::DomainError("exchange chunk must be a power of two");
        e->chunk_amps = static_cast<uint64_t>(amps);
    });
}

// ---------------------------------------------------------------- registers

Qureg createQureg(int numQubits, QuESTEnv env) {
    return guarded("createQureg", null_qureg(),
                   [&] { return make_handle(create_register(env_of(env), numQubits, false)); });
}

Qureg createDensityQureg(int numQubits, QuESTEnv env) {
    return guarded("createDensityQureg", null_qureg(),
                   [&] { return make_handle(create_register(env_of(env), numQubits, true)); });
}

Qureg qgpuCreateQuregPrecision(int numQubits, QuESTEnv env, int density, int precision) {
    return guarded("qgpuCreateQuregPrecision", null_qureg(), [&] {
        if (precision != 1 && precision != 2)
            throw qgpu::DomainError("precision must be 1 (single) or 2 (double), got " +
                                    std::to_string(precision));
        return make_handle(create_register(env_of(env), numQubits, density != 0, precision == 1));
    });
}

int qgpuGetPrecision(Qureg qureg) {
    return guarded("qgpuGetPrecision", -1, [&] { return reg_of(qureg)->single ? 1 : 2; });
}

Qureg createCloneQureg(Qureg qureg, QuESTEnv env) {
    return guarded("createCloneQureg", null_qureg(), [&] {
        QuregImpl* src = reg_of(qureg);
        if (env_of(env) != src->env) // shards are copied one to one (same ranks, same stream)
            throw qgpu::DomainError("createCloneQureg needs the environment the source register lives in");
        QuregImpl* r = create_register(env_of(env), src->N, src->density, src->single);
        src->flush();
        r->sp = src->sp; // same logical -> physical qubit map
        for (size_t k = 0; k < r->shards.size(); ++k)
            cuda_check(memcpy_counted(r->shards[k].amps, src->shards[k].amps,
                                       r->local_len * r->amp_bytes(), cudaMemcpyDeviceToDevice,
                                       src->env->stream),
                       "clone");
        cuda_check(cudaStreamSynchronize(src->env->stream), "clone");
        return make_handle(r);
    });
}

void destroyQureg(Qureg qureg, QuESTEnv env) {
    (void)env;
    guarded_void("destroyQureg", [&] {
        QuregImpl* r = reg_of(qureg);
        {
            std::lock_guard<std::mutex> lk(g_live_mu);
            g_live.erase(r);
        }
        delete r;
    });
}

int getNumQubits(Qureg qureg) {
    return guarded("getNumQubits", -1, [&] { return reg_of(qureg)->N; });
}

long long int getNumAmps(Qureg qureg) {
    return guarded("getNumAmps", -1LL, [&] {
        QuregImpl* r = reg_of(qureg);
        require_statevec(r, "getNumAmps");
        return static_cast<long long>(uint64_t{1} << r->flat);
    });
}

unsigned long long qgpuPassCount(Qureg qureg) {
    return guarded("qgpuPassCount", 0ULL, [&] { return static_cast<unsigned long long>(reg_of(qureg)->passes); });
}

void qgpuFlush(Qureg qureg) {
    guarded_void("qgpuFlush", [&] { reg_of(qureg)->flush(); });
}

void qgpuCommStats(Qureg qureg, unsigned long long* messages, unsigned long long* bytes) {
    guarded_void("qgpuCommStats", [&] {
        QuregImpl* r = reg_of(qureg);
        for (size_t k = 0; k < r->shards.size(); ++k) {
            if (messages) messages[k] = r->shards[k].messages;
            if (bytes) bytes[k] = r->shards[k].bytes;
        }
    });
}

// ------------------------------------------------------------ initialisers

void initZeroState(Qureg qureg) {
    guarded_void("initZeroState", [&] {
        QuregImpl* r = reg_of(qureg);
        r->fill_zero(); // queued ops are dead: discarded, not executed
        const double2 one = make_double2(1.0, 0.0);
        r->set_flat(0, 1, &one);
    });
}

void initPlusState(Qureg qureg) {
    guarded_void("initPlusState", [&] {
        QuregImpl* r = reg_of(qureg);
        r->discard_all(); // queued logical ops are dead too (lq), not just the open pass
        r->sp.reset(r->flat, r->local_qubits, r->env->swap_granule()); // uniform state: any layout
        const double v = r->density ? 1.0 / static_cast<double>(uint64_t{1} << r->N)
                                    : 1.0 / std::sqrt(static_cast<double>(uint64_t{1} << r->N));
        for (auto& s : r->shards) launch_fill(s.amps, r->single, r->local_len, v, 0.0, r->env->stream);
        cuda_check(cudaGetLastError(), "initPlusState");
    });
}

void initClassicalState(Qureg qureg, long long int stateInd) {
    guarded_void("initClassicalState", [&] {
        QuregImpl* r = reg_of(qureg);
        const uint64_t dim = uint64_t{1} << r->N;
        if (stateInd < 0 || static_cast<uint64_t>(stateInd) >= dim)
            throw qgpu::DomainError("invalid state index " + std::to_string(stateInd));
        r->fill_zero();
        const uint64_t flat = r->density ? static_cast<uint64_t>(stateInd) * (dim + 1)
                                         : static_cast<uint64_t>(stateInd);
        const double2 one = make_double2(1.0, 0.0);
        r->set_flat(flat, 1, &one);
    });
}

static void set_amps_impl(QuregImpl* r, long long start, const double* re, const double* im,
                          const double* inter, long long num) {
    const uint64_t len = uint64_t{1} << r->flat;
    if (num < 0 || start < 0 || static_cast<uint64_t>(start) > len ||
        static_cast<uint64_t>(num) > len - static_cast<uint64_t>(start))
        throw qgpu::DomainError("amplitude range [" + std::to_string(start) + ", " +
                                std::to_string(start + num) + ") out of range [0, " +
                                std::to_string(len) + ")");
    std::vector<double2> buf(static_cast<size_t>(num));
    for (long long i = 0; i < num; ++i) {
        const double x = inter ? inter[2 * i] : re[i];
        const double y = inter ? inter[2 * i + 1] : im[i];
        if (!std::isfinite(x) || !std::isfinite(y)) // register.cpp:46-47
            throw qgpu::DomainError("amplitude must be finite");
        buf[static_cast<size_t>(i)] = make_double2(x, y);
    }
    if (num) r->set_flat(static_cast<uint64_t>(start), static_cast<uint64_t>(num), buf.data());
}

void setAmps(Qureg qureg, long long int startInd, qreal* reals, qreal* imags,
             long long int numAmps) {
    guarded_void("setAmps", [&] {
        QuregImpl* r = reg_of(qureg);
        require_statevec(r, "setAmps");
        if (numAmps > 0 && (!reals || !imags)) throw qgpu::DomainError("null amplitude arrays");
        set_amps_impl(r, startInd, reals, imags, nullptr, numAmps);
    });
}

void initStateFromAmps(Qureg qureg, qreal* reals, qreal* imags) {
    guarded_void("initStateFromAmps", [&] {
        QuregImpl* r = reg_of(qureg);
        require_statevec(r, "initStateFromAmps");
        if (!reals || !imags) throw qgpu::DomainError("null amplitude arrays");
        const uint64_t len = uint64_t{1} << r->flat;
        for (uint64_t i = 0; i < len; ++i) // validate before any mutation (register.cpp:46-47)
            if (!std::isfinite(reals[i]) || !std::isfinite(imags[i]))
                throw qgpu::DomainError("amplitude must be finite");
        r->discard_all(); // the whole state is rewritten: drop queued ops and the qubit permutation
        r->sp.reset(r->flat, r->local_qubits, r->env->swap_granule());
        set_amps_impl(r, 0, reals, imags, nullptr, static_cast<long long>(uint64_t{1} << r->flat));
    });
}

void qgpuCopyStateFromHost(Qureg qureg, long long int start, long long int num, const double* in) {
    guarded_void("qgpuCopyStateFromHost", [&] {
        QuregImpl* r = reg_of(qureg);
        if (num > 0 && !in) throw qgpu::DomainError("null amplitude array");
        set_amps_impl(r, start, nullptr, nullptr, in, num);
    });
}

void qgpuCopyStateToHost(Qureg qureg, long long int start, long long int num, double* out) {
    guarded_void("qgpuCopyStateToHost", [&] {
        QuregImpl* r = reg_of(qureg);
        const uint64_t len = uint64_t{1} << r->flat;
        if (num < 0 || start < 0 || static_cast<uint64_t>(start) > len ||
            static_cast<uint64_t>(num) > len - static_cast<uint64_t>(start))
            throw qgpu::DomainError("amplitude range out of range [0, " + std::to_string(len) + ")");
        if (num > 0 && !out) throw qgpu::DomainError("null output array");
        if (num) r->get_flat(static_cast<uint64_t>(start), static_cast<uint64_t>(num),
                             reinterpret_cast<double2*>(out));
    });
}

void cloneQureg(Qureg targetQureg, Qureg copyQureg) {
    guarded_void("cloneQureg", [&] {
        QuregImpl* t = reg_of(targetQureg);
        QuregImpl* c = reg_of(copyQureg);
        if (t->density != c->density || t->N != c->N || t->env != c->env || t->single != c->single)
            throw qgpu::DomainError("cloneQureg needs registers of the same kind, size and precision");
        c->flush();
        t->discard_all();
        t->sp = c->sp;
        for (size_t k = 0; k < t->shards.size(); ++k)
            cuda_check(memcpy_counted(t->shards[k].amps, c->shards[k].amps,
                                       t->local_len * t->amp_bytes(), cudaMemcpyDeviceToDevice,
                                       t->env->stream),
                       "cloneQureg");
    });
}

// -------------------------------------------------------------- amplitudes

Complex getAmp(Qureg qureg, long long int index) {
    return guarded("getAmp", Complex{0, 0}, [&] {
        QuregImpl* r = reg_of(qureg);
        require_statevec(r, "getAmp");
        const double2 v = read_flat(r, index);
        return Complex{v.x, v.y};
    });
}

qreal getRealAmp(Qureg qureg, long long int index) { return getAmp(qureg, index).real; }
qreal getImagAmp(Qureg qureg, long long int index) { return getAmp(qureg, index).imag; }

qreal getProbAmp(Qureg qureg, long long int index) {
    const Complex c = getAmp(qureg, index);
    return c.real * c.real + c.imag * c.imag;
}

Complex getDensityAmp(Qureg qureg, long long int row, long long int col) {
    return guarded("getDensityAmp", Complex{0, 0}, [&] {
        QuregImpl* r = reg_of(qureg);
        require_density(r, "getDensityAmp");
        const long long dim = 1LL << r->N;
        if (row < 0 || row >= dim || col < 0 || col >= dim)
            throw qgpu::DomainError("invalid density-matrix element (" + std::to_string(row) +
                                    ", " + std::to_string(col) + ")");
        const double2 v = read_flat(r, row + dim * col); // register.hpp:47-50
        return Complex{v.x, v.y};
    });
}

// ------------------------------------------------------------------- gates

void hadamard(Qureg q, int t) { gate_call("hadamard", q, nullptr, 0, t, m_hadamard()); }
void pauliX(Qureg q, int t) { gate_call("pauliX", q, nullptr, 0, t, m_x()); }
void pauliY(Qureg q, int t) { gate_call("pauliY", q, nullptr, 0, t, m_y()); }
void pauliZ(Qureg q, int t) { gate_call("pauliZ", q, nullptr, 0, t, m_z()); }
void sGate(Qureg q, int t) { gate_call("sGate", q, nullptr, 0, t, m_s()); }
void tGate(Qureg q, int t) { gate_call("tGate", q, nullptr, 0, t, m_t()); }
void phaseShift(Qureg q, int t, qreal angle) {
    gate_call("phaseShift", q, nullptr, 0, t, m_phase(angle));
}
void rotateX(Qureg q, int t, qreal angle) {
    gate_call("rotateX", q, nullptr, 0, t, m_rotation(1, 0, 0, angle));
}
void rotateY(Qureg q, int t, qreal angle) {
    gate_call("rotateY", q, nullptr, 0, t, m_rotation(0, 1, 0, angle));
}
void rotateZ(Qureg q, int t, qreal angle) {
    gate_call("rotateZ", q, nullptr, 0, t, m_rotation(0, 0, 1, angle));
}
void rotateAroundAxis(Qureg q, int t, qreal angle, Vector axis) {
    guarded_void("rotateAroundAxis", [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, nullptr, 0, t);
        apply_gate(r, t, mask, m_axis(angle, axis));
    });
}
void compactUnitary(Qureg q, int t, Complex alpha, Complex beta) {
    guarded_void("compactUnitary", [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, nullptr, 0, t);
        apply_gate(r, t, mask, m_compact(alpha, beta));
    });
}
void unitary(Qureg q, int t, ComplexMatrix2 u) {
    guarded_void("unitary", [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, nullptr, 0, t);
        apply_gate(r, t, mask, checked_unitary(from_cm2(u)));
    });
}

void controlledNot(Qureg q, int c, int t) { gate_call("controlledNot", q, &c, 1, t, m_x()); }
void controlledPauliY(Qureg q, int c, int t) { gate_call("controlledPauliY", q, &c, 1, t, m_y()); }
void controlledPhaseFlip(Qureg q, int q1, int q2) {
    gate_call("controlledPhaseFlip", q, &q2, 1, q1, m_z());
}
void controlledPhaseShift(Qureg q, int q1, int q2, qreal angle) {
    gate_call("controlledPhaseShift", q, &q2, 1, q1, m_phase(angle));
}
void multiControlledPhaseFlip(Qureg q, int* ctrls, int n) {
    guarded_void("multiControlledPhaseFlip", [&] {
        if (n < 1 || !ctrls) throw qgpu::DomainError("need at least one qubit");
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, ctrls, n - 1, ctrls[n - 1]);
        apply_gate(r, ctrls[n - 1], mask, m_z());
    });
}
void multiControlledPhaseShift(Qureg q, int* ctrls, int n, qreal angle) {
    guarded_void("multiControlledPhaseShift", [&] {
        if (n < 1 || !ctrls) throw qgpu::DomainError("need at least one qubit");
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, ctrls, n - 1, ctrls[n - 1]);
        apply_gate(r, ctrls[n - 1], mask, m_phase(angle));
    });
}
void controlledRotateX(Qureg q, int c, int t, qreal angle) {
    gate_call("controlledRotateX", q, &c, 1, t, m_rotation(1, 0, 0, angle));
}
void controlledRotateY(Qureg q, int c, int t, qreal angle) {
    gate_call("controlledRotateY", q, &c, 1, t, m_rotation(0, 1, 0, angle));
}
void controlledRotateZ(Qureg q, int c, int t, qreal angle) {
    gate_call("controlledRotateZ", q, &c, 1, t, m_rotation(0, 0, 1, angle));
}
void controlledRotateAroundAxis(Qureg q, int c, int t, qreal angle, Vector axis) {
    guarded_void("controlledRotateAroundAxis", [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, &c, 1, t);
        apply_gate(r, t, mask, m_axis(angle, axis));
    });
}
void controlledCompactUnitary(Qureg q, int c, int t, Complex alpha, Complex beta) {
    guarded_void("controlledCompactUnitary", [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, &c, 1, t);
        apply_gate(r, t, mask, m_compact(alpha, beta));
    });
}
void controlledUnitary(Qureg q, int c, int t, ComplexMatrix2 u) {
    guarded_void("controlledUnitary", [&] {
        QuregImpl* r = reg_of(q);
        const uint64_t mask = control_mask(r, &c, 1, t);
        apply_gate(r, t, mask, checked_unitary(from_cm2(u)));
    });
}
void multiControlledUnitary(Qureg q, int* ctrls, int n, int t, ComplexMatrix2 u) {
    guarded_void("multiControlledUnitary", [&] {
        QuregImpl* r = reg_of(q);
        if (n < 0 || (n > 0 && !ctrls)) throw qgpu::DomainError("invalid control list");
        const uint64_t mask = control_mask(r, ctrls, n, t);
        apply_gate(r, t, mask, checked_unitary(from_cm2(u)));
    });
}

void qgpuApplyMatrix(Qureg q, int t, unsigned long long ctrlMask, const double* m8) {
    guarded_void("qgpuApplyMatrix", [&] {
        QuregImpl* r = reg_of(q);
        if (!m8) throw qgpu::DomainError("null matrix");
        std::vector<int> ctrls;
        for (int b = 0; b < 64; ++b)
            if ((ctrlMask >> b) & 1) {
                if (b >= r->N) {
                    if (r->density)
                        throw qgpu::DomainError("invalid qubit " + std::to_string(b) + " for " +
                                                std::to_string(r->N) + "-qubit density matrix");
                    throw qgpu::DomainError("invalid control qubit " + std::to_string(b));
                }
                ctrls.push_back(b);
            }
        const uint64_t mask = control_mask(r, ctrls.data(), static_cast<int>(ctrls.size()), t);
        M2 g;
        for (int k = 0; k < 8; ++k) {
            if (!std::isfinite(m8[k])) throw qgpu::DomainError("matrix entries must be finite");
            g.m[k] = m8[k];
        }
        apply_gate(r, t, mask, g);
    });
}

// ------------------------------------------------------------- measurement

qreal calcTotalProb(Qureg qureg) {
    return guarded("calcTotalProb", 0.0, [&] {
        QuregImpl* r = reg_of(qureg);
        return r->density ? r->reduce_diag(-1, 0) : r->reduce_norm(-1, 0);
    });
}

qreal qgpuNormSquared(Qureg qureg) {
    return guarded("qgpuNormSquared", 0.0, [&] { return reg_of(qureg)->reduce_norm(-1, 0); });
}

Complex qgpuTrace(Qureg qureg) {
    return guarded("qgpuTrace", Complex{0, 0}, [&] {
        QuregImpl* r = reg_of(qureg);
        require_density(r, "trace");
        return r->trace();
    });
}

qreal calcPurity(Qureg qureg) {
    return guarded("calcPurity", 0.0, [&] {
        QuregImpl* r = reg_of(qureg);
        require_density(r, "purity");
        return r->reduce_norm(-1, 0); // density.cpp:156-159
    });
}

qreal calcProbOfOutcome(Qureg qureg, int measureQubit, int outcome) {
    return guarded("calcProbOfOutcome", 0.0, [&] {
        QuregImpl* r = reg_of(qureg);
        check_qubit(r, measureQubit, "target");
        check_outcome(outcome);
        return prob_of_outcome(r, measureQubit, outcome);
    });
}

qreal collapseToOutcome(Qureg qureg, int measureQubit, int outcome) {
    return guarded("collapseToOutcome", 0.0, [&] {
        QuregImpl* r = reg_of(qureg);
        check_qubit(r, measureQubit, "target");
        check_outcome(outcome);
        const double p = prob_of_outcome(r, measureQubit, outcome);
        if (!(p > 1e-13))
            throw qgpu::DomainError("can't collapse to state with zero probability");
        enqueue_collapse(r, measureQubit, outcome, p);
        return p;
    });
}

int measureWithStats(Qureg qureg, int measureQubit, qreal* outcomeProb) {
    return guarded("measureWithStats", -1, [&] {
        QuregImpl* r = reg_of(qureg);
        check_qubit(r, measureQubit, "target");
        const double p0 = prob_of_outcome(r, measureQubit, 0);
        int outcome;
        if (p0 < 1e-13)
            outcome = 1;
        else if (1.0 - p0 < 1e-13)
            outcome = 0;
        else
            outcome = static_cast<double>(splitmix_next(&r->env->rng) >> 11) * 0x1.0p-53 > p0 ? 1 : 0;
        const double p = outcome == 0 ? p0 : prob_of_outcome(r, measureQubit, 1);
        enqueue_collapse(r, measureQubit, outcome, p);
        if (outcomeProb) *outcomeProb = p;
        return outcome;
    });
}

int measure(Qureg qureg, int measureQubit) {
    return measureWithStats(qureg, measureQubit, nullptr);
}

// ------------------------------------------------------------------- noise

void mixDephasing(Qureg qureg, int targetQubit, qreal prob) {
    guarded_void("mixDephasing", [&] {
        QuregImpl* r = reg_of(qureg);
        require_density(r, "dephasing");
        check_qubit(r, targetQubit, "target");
        if (!(prob >= 0.0 && prob <= 0.5)) // density.cpp:124-126
            throw qgpu::DomainError("dephasing probability must lie in [0, 1/2], got " +
                                    std::to_string(prob));
        FlatOp op;
        op.kind = FK_DEPHASE;
        op.q0 = targetQubit;
        op.q1 = targetQubit + r->N;
        op.m[0] = 1.0 - 2.0 * prob; // density.cpp:53
        r->enqueue(op);
    });
}

void mixDepolarising(Qureg qureg, int targetQubit, qreal prob) {
    guarded_void("mixDepolarising", [&] {
        QuregImpl* r = reg_of(qureg);
        require_density(r, "depolarising");
        check_qubit(r, targetQubit, "target");
        if (!(prob >= 0.0 && prob <= 0.75)) // density.cpp:137-140
            throw qgpu::DomainError("depolarising probability must lie in [0, 3/4], got " +
                                    std::to_string(prob));
        FlatOp op;
        op.kind = FK_DEPOL;
        op.q0 = targetQubit;
        op.q1 = targetQubit + r->N;
        op.m[0] = 1.0 - 2.0 * prob / 3.0; // density.cpp:70-72
        op.m[1] = 2.0 * prob / 3.0;
        op.m[2] = 1.0 - 4.0 * prob / 3.0;
        r->enqueue(op);
    });
}

// ------------------------------------------------------------ run_circuit

// circuit.cpp:239-247 (run_circuit) as one call: every op is validated with
// the rules of its single-op entry point before any is queued, so an invalid
// op leaves the register untouched; then the ops are queued in order.
void qgpuRunCircuit(Qureg qureg, const qgpuOp* ops, int numOps) {
    guarded_void("qgpuRunCircuit", [&] {
        QuregImpl* r = reg_of(qureg);
        if (numOps < 0 || (numOps > 0 && !ops)) throw qgpu::DomainError("invalid op array");
        std::vector<FlatOp> flat;
        flat.reserve(static_cast<size_t>(numOps) * (r->density ? 2 : 1));
        for (int i = 0; i < numOps; ++i) {
            const qgpuOp& o = ops[i];
            switch (o.kind) {
            case 0: { // gate: apply_controlled_gate / apply_gate_to_density
                check_qubit(r, o.target, "target");
                if (o.ctrlMask >> r->N) {
                    const int b = 63 - __builtin_clzll(o.ctrlMask);
                    if (r->density)
                        throw qgpu::DomainError("invalid qubit " + std::to_string(b) + " for " +
                                                std::to_string(r->N) + "-qubit density matrix");
                    throw qgpu::DomainError("invalid control qubit " + std::to_string(b));
                }
                if ((o.ctrlMask >> o.target) & 1)
                    throw qgpu::DomainError("control qubit " + std::to_string(o.target) + " overlaps the target");
                FlatOp op;
                op.kind = FK_GATE;
                op.q0 = o.target;
                op.cmask = o.ctrlMask;
                for (int k = 0; k < 8; ++k) {
                    if (!std::isfinite(o.m[k])) throw qgpu::DomainError("matrix entries must be finite");
                    op.m[k] = o.m[k];
                }
                op.cls = classify(op.m, &op.flags);
                flat.push_back(op);
                if (r->density) {
                    FlatOp bra = op;
                    bra.q0 = o.target + r->N;
                    bra.cmask = o.ctrlMask << r->N;
                    for (int k = 1; k < 8; k += 2) bra.m[k] = -op.m[k]; // GateMatrix::conjugate
                    bra.cls = classify(bra.m, &bra.flags);
                    flat.push_back(bra);
                }
                break;
            }
            case 1: { // apply_dephasing (density.cpp:118-130)
                require_density(r, "dephasing");
                check_qubit(r, o.target, "target");
                if (!(o.prob >= 0.0 && o.prob <= 0.5))
                    throw qgpu::DomainError("dephasing probability must lie in [0, 1/2], got " +
                                            std::to_string(o.prob));
                FlatOp op;
                op.kind = FK_DEPHASE;
                op.q0 = o.target;
                op.q1 = o.target + r->N;
                op.m[0] = 1.0 - 2.0 * o.prob;
                flat.push_back(op);
                break;
            }
            case 2: { // apply_depolarising (density.cpp:132-145)
                require_density(r, "depolarising");
                check_qubit(r, o.target, "target");
                if (!(o.prob >= 0.0 && o.prob <= 0.75))
                    throw qgpu::DomainError("depolarising probability must lie in [0, 3/4], got " +
                                            std::to_string(o.prob));
                FlatOp op;
                op.kind = FK_DEPOL;
                op.q0 = o.target;
                op.q1 = o.target + r->N;
                op.m[0] = 1.0 - 2.0 * o.prob / 3.0;
                op.m[1] = 2.0 * o.prob / 3.0;
                op.m[2] = 1.0 - 4.0 * o.prob / 3.0;
                flat.push_back(op);
                break;
            }
            default:
                throw qgpu::DomainError("unknown op kind " + std::to_string(o.kind) + " at op " +
                                        std::to_string(i));
            }
        }
        for (const FlatOp& op : flat) r->enqueue(op);
    });
}

// ------------------------------------------------------------- profiling

void qgpuProfileStart(QuESTEnv env) {
    guarded_void("qgpuProfileStart", [&] {
        Env* e = env_of(env);
        for (QuregImpl* q : e->quregs) q->flush();
        for (auto& r : e->prof) {
            e->event_pool.push_back(r.start);
            e->event_pool.push_back(r.stop);
        }
        e->prof.clear();
        e->profile = true;
    });
}

int qgpuProfileStop(QuESTEnv env, double* ms, int* kinds, int maxRecords) {
    return guarded("qgpuProfileStop", -1, [&] {
        Env* e = env_of(env);
        for (QuregImpl* q : e->quregs) q->flush();
        e->profile = false;
        cuda_check(cudaStreamSynchronize(e->stream), "qgpuProfileStop");
        const int n = static_cast<int>(e->prof.size());
        for (int i = 0; i < n && i < maxRecords; ++i) {
            float t = 0.f;
            cuda_check(cudaEventElapsedTime(&t, e->prof[i].start, e->prof[i].stop),
                       "cudaEventElapsedTime");
            if (ms) ms[i] = t;
            if (kinds) kinds[i] = e->prof[i].kind;
        }
        return n;
    });
}

int qgpuProfileInfo(QuESTEnv env, int* info, int maxRecords) {
    return guarded("qgpuProfileInfo", -1, [&] {
        Env* e = env_of(env);
        const int n = static_cast<int>(e->prof.size());
        for (int i = 0; i < n && i < maxRecords; ++i)
            if (info) info[i] = e->prof[i].info;
        return n;
    });
}

// --------------------------------------------------------------- planner

int qgpuPlanGate(int flatQubits, int rankLog2, int rank, int target, unsigned long long ctrlMask,
                 int* peer, int* ownLo, unsigned long long* lowMask) {
    int p = 0, o = 0;
    uint64_t lm = 0;
    const int r = plan_gate(flatQubits, rankLog2, rank, target, ctrlMask, &p, &o, &lm);
    if (peer) *peer = p;
    if (ownLo) *ownLo = o;
    if (lowMask) *lowMask = lm;
    return r;
}

int qgpuPlanChunks(unsigned long long localLen, unsigned long long chunkAmps,
                   unsigned long long* chunkLen) {
    if (localLen == 0 || chunkAmps == 0) return -1;
    const unsigned long long c = chunkAmps < localLen ? chunkAmps : localLen;
    if (chunkLen) *chunkLen = c;
    return static_cast<int>((localLen + c - 1) / c);
}

// ------------------------------------------------------------ memory plan

int qgpuModeledBytesPerRank(int numQubits, int rankLog2, int strategy, int singlePrecision,
                            unsigned long long blockAmps, unsigned long long* bytes) {
    return guarded("qgpuModeledBytesPerRank", -1, [&] {
        const uint64_t b = qgpu::modeled_bytes_per_rank(numQubits, rankLog2, strategy,
                                                        singlePrecision != 0, blockAmps);
        if (bytes) *bytes = b;
        return 0;
    });
}

int qgpuMaxQubits(unsigned long long nodeBytes, unsigned long long overheadBytes, int strategy,
                  int singlePrecision, int rankLog2) {
    return guarded("qgpuMaxQubits", -1, [&] {
        return qgpu::max_qubits(nodeBytes, overheadBytes, strategy, singlePrecision != 0, rankLog2);
    });
}

unsigned long long qgpuDeviceBytesPerRank(int flatQubits, int rankLog2, unsigned long long chunkAmps,
                                          int singlePrecision) {
    return guarded("qgpuDeviceBytesPerRank", 0ull, [&] {
        return static_cast<unsigned long long>(
            qgpu::device_bytes_per_rank(flatQubits, rankLog2, chunkAmps, singlePrecision != 0));
    });
}

int qgpuDeviceMaxQubits(unsigned long long deviceBytes, int rankLog2, unsigned long long chunkAmps,
                        int density, int singlePrecision) {
    return guarded("qgpuDeviceMaxQubits", -1, [&] {
        return qgpu::device_max_qubits(deviceBytes, rankLog2, chunkAmps, density != 0, singlePrecision != 0);
    });
}

int qgpuPlanPasses(int flatQubits, int numOps, const int* kinds, const int* q0, const int* q1,
                   const unsigned long long* cmasks, const double* mats, int reorder, int windowOps,
                   int maxPhases, int* orderOut, int* passOut, int* phaseOut) {
    return guarded("qgpuPlanPasses", -1, [&] {
        if (flatQubits < kTileQubits || flatQubits > 62 || numOps < 0 || maxPhases < 1 || maxPhases > kMaxPhases)
            throw qgpu::DomainError("invalid pass-plan request");
        Env e;
        if (const char* v = std::getenv("QGPU_LANE_CAP")) e.lane_cap = std::max(0, std::atoi(v));
        if (const char* v = std::getenv("QGPU_XCHG")) e.exchanges = std::atoi(v);
        if (const char* v = std::getenv("QGPU_MERGE")) e.merge = std::atoi(v) != 0;
        if (const char* v = std::getenv("QGPU_SWIZZLE")) e.swizzle = std::max(0, std::atoi(v));
        e.order = reorder ? 1 : 0;
        if (windowOps > 0) e.window = windowOps;
        e.tile_phases = maxPhases;
        QuregImpl q;
        q.N = q.flat = flatQubits;
        q.local_qubits = flatQubits;
        q.local_len = uint64_t{1} << flatQubits;
        std::vector<QuregImpl::PlannedPass> out;
        q.plan_sink = &out;
        q.env = &e;
        try {
            for (int i = 0; i < numOps; ++i) {
                FlatOp op;
                op.kind = static_cast<uint8_t>(kinds[i]);
                op.q0 = q0[i];
                op.q1 = q1[i];
                op.cmask = cmasks[i];
                op.id = i;
                if (op.q0 < 0 || op.q0 >= flatQubits || op.q1 >= flatQubits || (op.cmask >> flatQubits))
                    throw qgpu::DomainError("op " + std::to_string(i) + " out of range");
                if (op.kind == FK_GATE) {
                    std::memcpy(op.m, mats + 8 * static_cast<size_t>(i), sizeof(op.m));
                    op.cls = classify(op.m, &op.flags);
                } else if (op.kind > FK_COLLAPSE) {
                    throw qgpu::DomainError("op " + std::to_string(i) + ": unknown kind");
                }
                q.enqueue_phys(op);
            }
            q.flush_pass();
        } catch (...) {
            q.env = nullptr;
            throw;
        }
        q.env = nullptr;
        int k = 0;
        for (size_t p = 0; p < out.size(); ++p) {
            const auto& pp = out[p];
            for (size_t j = 0; j < pp.ids.size(); ++j) {
                if (pp.ids[j] < 0) continue; // the scheduler's own ops (a folded-out scalar)
                int ph = 0;
                while (ph + 1 < static_cast<int>(pp.phase_begin.size()) && pp.phase_begin[ph + 1] <= static_cast<int>(j)) ++ph;
                if (k >= numOps) throw qgpu::DeviceError("internal: plan has more ops than the input");
                orderOut[k] = pp.ids[j];
                passOut[k] = static_cast<int>(p);
                phaseOut[k] = ph;
                ++k;
            }
        }
        if (k != numOps) throw qgpu::DeviceError("internal: plan lost ops");
        return static_cast<int>(out.size());
    });
}

int qgpuPlanDistributed(int flatQubits, int rankLog2, int numOps, const int* kinds, const int* q0, const int* q1,
                        const unsigned long long* cmasks, const double* mats, int reorder, int* passesOut,
                        int* swapsOut, int maxSwaps) {
    return guarded("qgpuPlanDistributed", -1, [&] {
        if (rankLog2 < 1 || rankLog2 > 16 || flatQubits - rankLog2 < kTileQubits || flatQubits > 62 || numOps < 0 ||
            maxSwaps < 0)
            throw qgpu::DomainError("invalid distributed-plan request");
        Env e;
        e.mode = Mode::Peer; // (the swap granule of the peer transport; nothing is launched)
        e.rank_log2 = rankLog2;
        e.num_ranks = 1 << rankLog2;
        e.qubit_swaps = true;
        e.order = reorder ? 1 : 0;
        e.tile_phases = 3; // as on the GPU with the per-pass JIT (the host has no driver to JIT with)
        QuregImpl q;
        q.N = q.flat = flatQubits;
        q.local_qubits = flatQubits - rankLog2;
        q.local_len = uint64_t{1} << q.local_qubits;
        q.env = &e;
        q.sp.reset(q.flat, q.local_qubits, e.swap_granule());
        std::vector<QuregImpl::PlannedPass> out;
        std::vector<std::pair<int, int>> swaps;
        q.plan_sink = &out;
        q.swap_sink = &swaps;
        try {
            for (int i = 0; i < numOps; ++i) {
                FlatOp op;
                op.kind = static_cast<uint8_t>(kinds[i]);
                op.q0 = q0[i];
                op.q1 = q1[i];
                op.cmask = cmasks[i];
                op.id = i;
                if (op.q0 < 0 || op.q0 >= flatQubits || op.q1 >= flatQubits || (op.cmask >> flatQubits))
                    throw qgpu::DomainError("op " + std::to_string(i) + " out of range");
                if (op.kind == FK_GATE) {
                    std::memcpy(op.m, mats + 8 * static_cast<size_t>(i), sizeof(op.m));
                    op.cls = classify(op.m, &op.flags);
                } else if (op.kind > FK_COLLAPSE) {
                    throw qgpu::DomainError("op " + std::to_string(i) + ": unknown kind");
                }
                q.enqueue(op);
            }
            q.flush();
        } catch (...) {
            q.env = nullptr;
            throw;
        }
        q.env = nullptr;
        *passesOut = static_cast<int>(out.size());
        for (size_t i = 0; i < swaps.size() && static_cast<int>(i) < maxSwaps; ++i) {
            swapsOut[2 * i] = swaps[i].first;
            swapsOut[2 * i + 1] = swaps[i].second;
        }
        return static_cast<int>(swaps.size());
    });
}

void qgpuSetOrdering(QuESTEnv env, int reorder, int windowOps) {
    guarded_void("qgpuSetOrdering", [&] {
        Env* e = env_of(env);
        if (reorder != 0 && reorder != 1) throw qgpu::DomainError("ordering must be 0 (circuit order) or 1 (reorder)");
        if (windowOps < 0 || windowOps > 65536) throw qgpu::DomainError("reorder window must be 0..65536 ops");
        for (QuregImpl* q : e->quregs) q->flush();
        e->order = reorder;
        if (windowOps > 0) e->window = windowOps;
    });
}

int qgpuGetOrdering(QuESTEnv env) {
    return guarded("qgpuGetOrdering", -1, [&] { return env_of(env)->order; });
}

void qgpuSetQubitSwaps(QuESTEnv env, int enable) {
    guarded_void("qgpuSetQubitSwaps", [&] {
        Env* e = env_of(env);
        for (QuregImpl* q : e->quregs) q->restore_identity();
        e->qubit_swaps = enable != 0;
    });
}

int qgpuPlanSwaps(int flatQubits, int rankLog2, unsigned long long chunkAmps, int numOps,
                  const int* targets, const int* pairOps, int* swapsOut, int maxSwaps) {
    return guarded("qgpuPlanSwaps", -1, [&] {
        if (flatQubits < 1 || rankLog2 < 1 || rankLog2 >= flatQubits || numOps < 0)
            throw qgpu::DomainError("invalid swap-plan request");
        qgpu::SwapPlanner sp;
        const int local = flatQubits - rankLog2;
        sp.reset(flatQubits, local, chunkAmps);
        std::vector<int> need(static_cast<size_t>(numOps), -1);
        for (int k = 0; k < numOps; ++k) {
            if (targets[k] < 0 || targets[k] >= flatQubits) throw qgpu::DomainError("target out of range");
            if (pairOps[k]) need[k] = targets[k]; // diagonal ops never move
        }
        // the runtime's windowing (QuregImpl::enqueue / drain): ops are
        // planned when kSwapWindow are buffered (the first half) or at a flush
        int n = 0;
        size_t begin = 0, end = 0;
        const size_t total = static_cast<size_t>(numOps);
        while (begin < total) {
            end = std::min(total, begin + qgpu::kSwapWindow);
            const size_t count = end == total ? end - begin : qgpu::kSwapWindow / 2;
            for (size_t i = begin; i < begin + count; ++i) {
                if (need[i] < 0) continue;
                sp.touch(need[i]);
                const int p = sp.l2p[need[i]];
                if (p < local) continue;
                const int v = sp.victim(0, need.data() + i + 1, nullptr, end - i - 1);
                if (swapsOut && n < maxSwaps) {
                    swapsOut[3 * n] = static_cast<int>(i);
                    swapsOut[3 * n + 1] = p;
                    swapsOut[3 * n + 2] = v;
                }
                sp.apply(p, v);
                ++n;
            }
            begin += count;
        }
        return n;
    });
}

// ------------------------------------------------------------ per-pass JIT

void qgpuSetJit(int mode) {
    guarded_void("qgpuSetJit", [&] {
        if (mode < 0 || mode > 2) throw qgpu::DomainError("JIT mode must be 0 (off), 1 (background) or 2 (sync)");
        qgpu::jit_set_mode(mode);
    });
}

int qgpuGetJit(void) { return qgpu::jit_mode(); }

void qgpuJitWait(void) {
    guarded_void("qgpuJitWait", [&] { qgpu::jit_wait(); });
}

void qgpuJitShutdown(void) {
    guarded_void("qgpuJitShutdown", [&] { qgpu::jit_shutdown(); });
}

void qgpuJitStats(unsigned long long* kernels, unsigned long long* failed, unsigned long long* pending) {
    qgpu::jit_stats(kernels, failed, pending);
}

int qgpuJitSelfTest(char* log, int len, double* seconds) { return qgpu::jit_selftest(log, len, seconds); }

unsigned long long qgpuLaneExchanges(void) { return qgpu::g_lane_exchanges.load(); }

} // extern "C"
