// transport.h — NCCL transport (one process per GPU).
#pragma once

#include "runtime.h"

namespace qgpu {

class NcclComm {
  public:
    static void unique_id(char* out128);
    NcclComm(int rank, int nranks, const char* id128);
    ~NcclComm();
    NcclComm(const NcclComm&) = delete;
    NcclComm& operator=(const NcclComm&) = delete;

    void sendrecv(int peer, const void* send, void* recv, size_t bytes, cudaStream_t s);
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s);
    // ncclCommGetAsyncError: throws CommError (after aborting the
    // communicator) if NCCL reported an asynchronous failure
    void check_async();
    // ncclCommAbort: unblocks this rank's pending NCCL work (idempotent)
    void abort();
    int rank() const { return rank_; }
    int size() const { return nranks_; }

  private:
    void* comm_ = nullptr;
    int rank_ = 0, nranks_ = 1;
};

} // namespace qgpu
