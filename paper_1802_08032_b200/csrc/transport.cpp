// transport.cpp — NCCL point-to-point transport for the distributed engine,
// the B200 replacement of the reference's Transport::exchange / barrier
// (/root/reference/proj/include/qsim/transport.hpp:18-31).
//
// libnccl is resolved at run time: the copy already mapped into the process
// (torch's) if there is one, else the system libnccl.so.2. Only the handful
// of entry points the engine needs are bound, with their public C signatures.
#include "transport.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

namespace qgpu {

namespace {

using ncclComm_t = void*;
struct ncclUniqueId {
    char internal[128];
};
using ncclResult_t = int;
constexpr int ncclUint8 = 1;

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            a.handle = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
            if (a.handle) break;
        }
        if (!a.handle)
            for (const char* n : names) {
                a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
                if (a.handle) break;
            }
        if (!a.handle) return;
#define QGPU_BIND(field, sym) a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.handle, sym))
        QGPU_BIND(GetUniqueId, "ncclGetUniqueId");
        QGPU_BIND(CommInitRank, "ncclCommInitRank");
        QGPU_BIND(CommDestroy, "ncclCommDestroy");
        QGPU_BIND(CommAbort, "ncclCommAbort");
        QGPU_BIND(CommGetAsyncError, "ncclCommGetAsyncError");
        QGPU_BIND(Send, "ncclSend");
        QGPU_BIND(Recv, "ncclRecv");
        QGPU_BIND(AllGather, "ncclAllGather");
        QGPU_BIND(GroupStart, "ncclGroupStart");
        QGPU_BIND(GroupEnd, "ncclGroupEnd");
        QGPU_BIND(GetErrorString, "ncclGetErrorString");
#undef QGPU_BIND
    });
    if (!a.handle || !a.GetUniqueId || !a.CommInitRank || !a.Send || !a.Recv)
        throw CommError("NCCL is not available in this process (libnccl.so.2 not found)");
    return a;
}

void nccl_check(ncclResult_t r, const char* what, int rank, int peer) {
    if (r == 0) return;
    std::string msg = std::string(what) + " failed between ranks " + std::to_string(rank) +
                      " and " + std::to_string(peer);
    if (api().GetErrorString) msg += ": " + std::string(api().GetErrorString(r));
    throw CommError(msg);
}

} // namespace

void NcclComm::unique_id(char* out128) {
    ncclUniqueId id;
    nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId", -1, -1);
    std::memcpy(out128, id.internal, 128);
}

NcclComm::NcclComm(int rank, int nranks, const char* id128) : rank_(rank), nranks_(nranks) {
    ncclUniqueId id;
    std::memcpy(id.internal, id128, 128);
    nccl_check(api().CommInitRank(&comm_, nranks, id, rank), "ncclCommInitRank", rank, -1);
}

NcclComm::~NcclComm() {
    if (comm_ && api().CommDestroy) api().CommDestroy(comm_);
}

void NcclComm::abort() {
    if (comm_ && api().CommAbort) api().CommAbort(comm_);
    comm_ = nullptr;
}

void NcclComm::check_async() {
    if (!comm_) throw CommError("NCCL communicator of rank " + std::to_string(rank_) + " was aborted");
    if (!api().CommGetAsyncError) return;
    ncclResult_t st = 0;
    const ncclResult_t r = api().CommGetAsyncError(comm_, &st);
    constexpr ncclResult_t kInProgress = 7; // ncclInProgress
    if (r != 0 || (st != 0 && st != kInProgress)) {
        std::string msg = "NCCL asynchronous error on rank " + std::to_string(rank_);
        if (api().GetErrorString) msg += ": " + std::string(api().GetErrorString(r != 0 ? r : st));
        abort();
        throw CommError(msg);
    }
}

// One rendezvous exchange (transport.cpp:25-57 semantics: both sides send
// `bytes` and receive the peer's) as a grouped send/recv on `s`.
void NcclComm::sendrecv(int peer, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    auto& a = api();
    if (!comm_) throw CommError("NCCL communicator of rank " + std::to_string(rank_) + " was aborted");
    nccl_check(a.GroupStart(), "ncclGroupStart", rank_, peer);
    nccl_check(a.Send(send, bytes, ncclUint8, peer, comm_, s), "ncclSend", rank_, peer);
    nccl_check(a.Recv(recv, bytes, ncclUint8, peer, comm_, s), "ncclRecv", rank_, peer);
    nccl_check(a.GroupEnd(), "ncclGroupEnd", rank_, peer);
}

void NcclComm::allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) {
    if (!comm_) throw CommError("NCCL communicator of rank " + std::to_string(rank_) + " was aborted");
    nccl_check(api().AllGather(send, recv, bytes, ncclUint8, comm_, s), "ncclAllGather", rank_, -1);
}

} // namespace qgpu
