// peer.h — single-node peer-memory transport (one process per GPU).
//
// The B200 replacement of the reference's Transport (transport.hpp:18-62,
// InProcessTransport::exchange / barrier, transport.cpp:25-59) for one node of
// NVSwitch-connected GPUs: every rank maps every other rank's amplitude
// partition into its address space (CUDA IPC over NVLink), so an exchange
// gate or a global<->local qubit swap is ONE kernel that reads the partner's
// half and writes both halves in place — no staging buffer, no send/recv, no
// copy back (SURVEY.md §7 hard part 1; distributed.cpp:174-187's combine with
// each amplitude pair updated by exactly one GPU).
//
// Control plane (host): a POSIX shared-memory segment created by rank 0's
// qgpuPeerUniqueId holds
//   * a generation barrier (spin, then yield, then sleep) that fails with a
//     CommError instead of hanging when a peer process exited (pid liveness),
//     another rank aborted (its error message is carried), or
//     QGPU_PEER_TIMEOUT_S passed;
//   * double-buffered 128-byte mailboxes per rank for small all-gathers
//     (IPC handles, reduction partials, single amplitudes, the RNG seed).
// Stream ordering across processes uses interprocess CUDA events: a "fence"
// records this rank's event on its stream, passes the host barrier, and makes
// the stream wait on the partner ranks' events, so the GPU never spins.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace qgpu {

constexpr int kMaxPeers = 64;
constexpr int kPeerSlot = 1024; // bytes per rank per mailbox (a marginal vector: 37 x 16 B)

struct PeerShm; // peer.cpp

class PeerGroup {
  public:
    // Creates the shared segment; `out128` = its name (NUL-terminated).
    static void unique_id(char* out128);
    // with_cuda = false attaches the host control plane only (no device,
    // events or mappings: qgpuPeerProbe's self test)
    PeerGroup(int rank, int nranks, int device, const char* id128, bool with_cuda = true);
    ~PeerGroup();
    PeerGroup(const PeerGroup&) = delete;
    PeerGroup& operator=(const PeerGroup&) = delete;

    int rank() const { return rank_; }
    int size() const { return nranks_; }

    // host barrier over all ranks (CommError on a dead / aborted peer or
    // timeout)
    void barrier();
    // every rank contributes `bytes` (<= kPeerSlot); out[r * bytes] = rank r's
    void allgather(const void* in, void* out, size_t bytes);
    // mark the group failed (peers waiting in a barrier get CommError(msg))
    void abort(const std::string& msg);
    bool aborted() const;

    // Stream fence: record this rank's event on `s`, host barrier, then `s`
    // waits on the events of `wait_ranks` (their streams' work issued before
    // their own fence). Every rank calls it (SPMD), with its own wait list.
    void fence(cudaStream_t s, const std::vector<int>& wait_ranks);

    // Collective: maps every rank's device buffer. ptrs[r] = rank r's buffer
    // in this process (ptrs[rank] = mine). close_all unmaps (collective).
    std::vector<void*> open_all(void* mine);
    void close_all(std::vector<void*>& ptrs);

  private:
    int rank_ = 0, nranks_ = 1, device_ = 0;
    PeerShm* shm_ = nullptr;
    size_t shm_bytes_ = 0;
    std::string name_;
    uint64_t coll_seq_ = 0;  // all-gather mailbox parity
    uint64_t fence_seq_ = 0; // event parity
    cudaEvent_t events_[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> peer_events_[2];
    double timeout_s_ = 600.0;
};

} // namespace qgpu
