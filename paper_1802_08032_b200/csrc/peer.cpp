// peer.cpp — see peer.h. Host control plane of the single-node peer-memory
// transport: shared-memory barrier + mailboxes, interprocess CUDA events and
// IPC mappings of the ranks' partitions.
#include "peer.h"

#include "runtime.h"

#include <fcntl.h>
#include <sched.h>
#include <signal.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>

namespace qgpu {

namespace {
constexpr uint64_t kMagic = 0x71677075'70656572ull; // "qgpupeer"

// false once the process is gone or a zombie (exited, not yet reaped)
bool process_alive(int32_t pid) {
    if (kill(pid, 0) != 0) return errno != ESRCH;
    char path[64], buf[256];
    std::snprintf(path, sizeof(path), "/proc/%d/stat", static_cast<int>(pid));
    FILE* f = std::fopen(path, "r");
    if (!f) return true;
    const size_t n = std::fread(buf, 1, sizeof(buf) - 1, f);
    std::fclose(f);
    buf[n] = 0;
    const char* rp = std::strrchr(buf, ')'); // "pid (comm) S ..."
    return !(rp && rp[1] == ' ' && (rp[2] == 'Z' || rp[2] == 'X'));
}
} // namespace

struct PeerShm {
    uint64_t magic;
    std::atomic<int32_t> nranks;
    std::atomic<int32_t> attached;
    std::atomic<int32_t> abort_flag;
    char abort_msg[512];
    alignas(64) std::atomic<uint32_t> count;
    alignas(64) std::atomic<uint32_t> gen;
    alignas(64) std::atomic<int32_t> pids[kMaxPeers];
    alignas(64) unsigned char slots[2][kMaxPeers][kPeerSlot];
};

static_assert(std::atomic<uint32_t>::is_always_lock_free, "shared-memory atomics must be lock free");

void PeerGroup::unique_id(char* out128) {
    std::random_device rd;
    const uint64_t nonce = (static_cast<uint64_t>(rd()) << 32) ^ rd();
    char name[128];
    std::snprintf(name, sizeof(name), "/qgpu-peer-%d-%016llx", static_cast<int>(getpid()),
                  static_cast<unsigned long long>(nonce));
    const int fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw CommError(std::string("shm_open(") + name + "): " + std::strerror(errno));
    const size_t bytes = sizeof(PeerShm);
    if (ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
        close(fd);
        shm_unlink(name);
        throw CommError(std::string("ftruncate(") + name + "): " + std::strerror(errno));
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) {
        shm_unlink(name);
        throw CommError(std::string("mmap(") + name + "): " + std::strerror(errno));
    }
    auto* s = new (p) PeerShm; // ftruncate zero-filled it; atomics start at 0
    std::atomic_thread_fence(std::memory_order_release);
    s->magic = kMagic;
    munmap(p, bytes);
    std::memset(out128, 0, 128);
    std::strncpy(out128, name, 127);
}

PeerGroup::PeerGroup(int rank, int nranks, int device, const char* id128, bool with_cuda)
    : rank_(rank), nranks_(nranks), device_(device) {
    if (rank < 0 || rank >= nranks) throw DomainError("invalid rank " + std::to_string(rank));
    if (nranks < 1 || nranks > kMaxPeers)
        throw DomainError("peer group of " + std::to_string(nranks) + " ranks (max " +
                          std::to_string(kMaxPeers) + ")");
    if (const char* v = std::getenv("QGPU_PEER_TIMEOUT_S")) timeout_s_ = std::max(1.0, std::atof(v));
    char name[129];
    std::memcpy(name, id128, 128);
    name[128] = 0;
    name_ = name;
    const int fd = shm_open(name, O_RDWR, 0600);
    if (fd < 0)
        throw CommError("peer group " + name_ + " not found (" + std::strerror(errno) +
                        "): rank 0 creates it with qgpuPeerUniqueId");
    shm_bytes_ = sizeof(PeerShm);
    void* p = mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw CommError("mmap of the peer group failed: " + std::string(std::strerror(errno)));
    shm_ = static_cast<PeerShm*>(p);
    if (shm_->magic != kMagic) throw CommError("peer group " + name_ + " is not initialised");
    int32_t expect = 0;
    if (!shm_->nranks.compare_exchange_strong(expect, nranks) && expect != nranks)
        throw CommError("peer group " + name_ + " has " + std::to_string(expect) + " ranks, not " +
                        std::to_string(nranks));
    shm_->pids[rank].store(static_cast<int32_t>(getpid()));
    shm_->attached.fetch_add(1);
    try {
        barrier(); // everyone attached
        if (rank == 0) shm_unlink(name_.c_str());
        if (!with_cuda) return;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        // interprocess events for stream fences, two by parity
        cudaIpcEventHandle_t mine[2], all[2][kMaxPeers];
        for (int k = 0; k < 2; ++k) {
            cuda_check(cudaEventCreateWithFlags(&events_[k], cudaEventDisableTiming | cudaEventInterprocess),
                       "cudaEventCreate(interprocess)");
            cuda_check(cudaIpcGetEventHandle(&mine[k], events_[k]), "cudaIpcGetEventHandle");
        }
        static_assert(sizeof(cudaIpcEventHandle_t) * 2 <= kPeerSlot, "mailbox too small");
        std::vector<unsigned char> buf(static_cast<size_t>(nranks) * sizeof(mine));
        allgather(mine, buf.data(), sizeof(mine));
        for (int k = 0; k < 2; ++k) {
            peer_events_[k].assign(nranks, nullptr);
            for (int r = 0; r < nranks; ++r) {
                std::memcpy(&all[k][r], buf.data() + r * sizeof(mine) + k * sizeof(cudaIpcEventHandle_t),
                            sizeof(cudaIpcEventHandle_t));
                if (r == rank) {
                    peer_events_[k][r] = events_[k];
                    continue;
                }
                cuda_check(cudaIpcOpenEventHandle(&peer_events_[k][r], all[k][r]), "cudaIpcOpenEventHandle");
            }
        }
        barrier();
    } catch (const std::exception& e) {
        abort(std::string("rank ") + std::to_string(rank) + ": " + e.what());
        if (rank == 0) shm_unlink(name_.c_str());
        for (int k = 0; k < 2; ++k) {
            for (int r = 0; r < static_cast<int>(peer_events_[k].size()); ++r)
                if (r != rank && peer_events_[k][r]) cudaEventDestroy(peer_events_[k][r]);
            if (events_[k]) cudaEventDestroy(events_[k]);
        }
        munmap(shm_, shm_bytes_);
        shm_ = nullptr;
        throw;
    }
}

PeerGroup::~PeerGroup() {
    if (!shm_) return;
    if (!aborted()) {
        try {
            barrier(); // nobody still waits on our events
        } catch (...) {
        }
    }
    for (int k = 0; k < 2; ++k) {
        for (int r = 0; r < static_cast<int>(peer_events_[k].size()); ++r)
            if (r != rank_ && peer_events_[k][r]) cudaEventDestroy(peer_events_[k][r]);
        if (events_[k]) cudaEventDestroy(events_[k]);
    }
    munmap(shm_, shm_bytes_);
}

bool PeerGroup::aborted() const { return shm_ && shm_->abort_flag.load(std::memory_order_acquire) != 0; }

void PeerGroup::abort(const std::string& msg) {
    if (!shm_) return;
    int32_t expect = 0;
    if (shm_->abort_flag.compare_exchange_strong(expect, 2)) {
        std::strncpy(shm_->abort_msg, msg.c_str(), sizeof(shm_->abort_msg) - 1);
        shm_->abort_flag.store(1, std::memory_order_release);
    }
}

void PeerGroup::barrier() {
    auto failed = [&]() -> std::string {
        return std::string("peer group aborted: ") +
               (shm_->abort_flag.load(std::memory_order_acquire) == 1 ? shm_->abort_msg : "(in progress)");
    };
    if (aborted()) throw CommError(failed());
    const uint32_t g = shm_->gen.load(std::memory_order_acquire);
    if (shm_->count.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(nranks_)) {
        shm_->count.store(0, std::memory_order_relaxed);
        shm_->gen.store(g + 1, std::memory_order_release);
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    auto next_check = t0;
    for (uint64_t it = 0;; ++it) {
        if (shm_->gen.load(std::memory_order_acquire) != g) return;
        if (it < 2000) {
#if defined(__x86_64__)
            __builtin_ia32_pause();
#endif
            continue;
        }
        const auto now = std::chrono::steady_clock::now();
        if (now >= next_check) {
            next_check = now + std::chrono::milliseconds(10);
            if (aborted()) throw CommError(failed());
            for (int r = 0; r < nranks_; ++r) {
                const int32_t pid = shm_->pids[r].load(std::memory_order_relaxed);
                if (pid > 0 && r != rank_ && !process_alive(pid)) {
                    const std::string m = "rank " + std::to_string(r) + " (pid " + std::to_string(pid) +
                                          ") exited while rank " + std::to_string(rank_) +
                                          " waited in a barrier";
                    abort(m);
                    throw CommError(m);
                }
            }
            if (std::chrono::duration<double>(now - t0).count() > timeout_s_) {
                const std::string m = "rank " + std::to_string(rank_) + " timed out after " +
                                      std::to_string(static_cast<int>(timeout_s_)) +
                                      " s in a peer barrier (QGPU_PEER_TIMEOUT_S)";
                abort(m);
                throw CommError(m);
            }
        }
        if (it < 20000)
            sched_yield();
        else
            std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

void PeerGroup::allgather(const void* in, void* out, size_t bytes) {
    if (bytes > static_cast<size_t>(kPeerSlot)) throw DomainError("peer all-gather item too large");
    const int par = static_cast<int>(coll_seq_++ & 1);
    std::memcpy(shm_->slots[par][rank_], in, bytes);
    barrier(); // acq_rel on the barrier word publishes the slot
    for (int r = 0; r < nranks_; ++r)
        std::memcpy(static_cast<unsigned char*>(out) + static_cast<size_t>(r) * bytes, shm_->slots[par][r], bytes);
}

void PeerGroup::fence(cudaStream_t s, const std::vector<int>& wait_ranks) {
    const int par = static_cast<int>(fence_seq_++ & 1);
    cuda_check(cudaEventRecord(events_[par], s), "peer fence record");
    barrier();
    for (int r : wait_ranks)
        if (r != rank_) cuda_check(cudaStreamWaitEvent(s, peer_events_[par][r], 0), "peer fence wait");
}

std::vector<void*> PeerGroup::open_all(void* mine) {
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) <= kPeerSlot, "mailbox too small");
    cuda_check(cudaIpcGetMemHandle(&h, mine), "cudaIpcGetMemHandle");
    std::vector<cudaIpcMemHandle_t> all(nranks_);
    allgather(&h, all.data(), sizeof(h));
    std::vector<void*> ptrs(nranks_, nullptr);
    ptrs[rank_] = mine;
    for (int r = 0; r < nranks_; ++r) {
        if (r == rank_) continue;
        cuda_check(cudaIpcOpenMemHandle(&ptrs[r], all[r], cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
    }
    barrier();
    return ptrs;
}

void PeerGroup::close_all(std::vector<void*>& ptrs) {
    if (!aborted()) {
        try {
            barrier(); // no rank still reads or writes a peer's buffer
        } catch (...) {
        }
    }
    for (int r = 0; r < static_cast<int>(ptrs.size()); ++r)
        if (r != rank_ && ptrs[r]) cudaIpcCloseMemHandle(ptrs[r]);
    ptrs.clear();
    if (!aborted()) {
        try {
            barrier(); // every importer unmapped before the owner frees
        } catch (...) {
        }
    }
}

} // namespace qgpu
