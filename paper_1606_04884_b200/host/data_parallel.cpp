// data_parallel.cpp — batch-sharded data parallelism over NCCL for the C++ operator API
// (include/portten/data_parallel.hpp).
#include "portten/data_parallel.hpp"

#include <nccl.h>

#include <chrono>
#include <cstring>
#include <string>
#include <thread>

#include "portten/errors.hpp"

namespace portten {
void throw_if_error(int status);  // core.cpp
}

namespace portten::dp {

namespace {
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw BackendError(std::string("nccl: ") + what + ": " + ncclGetErrorString(r));
}
ncclComm_t as_comm(void* c) { return static_cast<ncclComm_t>(c); }
}  // namespace

ShardRange shard_range(std::int64_t n, int rank, int world) {
    PORTTEN_CHECK(world >= 1 && rank >= 0 && rank < world,
                  "shard_range: bad rank " + std::to_string(rank) + " for world size " + std::to_string(world));
    PORTTEN_CHECK(n >= 0, "shard_range: negative batch");
    const std::int64_t base = n / world, extra = n % world;
    const std::int64_t start = rank * base + (rank < extra ? rank : extra);
    return {start, start + base + (rank < extra ? 1 : 0)};
}

UniqueId new_unique_id() {
    static_assert(sizeof(ncclUniqueId) == sizeof(UniqueId), "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    UniqueId out;
    std::memcpy(out.data(), &id, sizeof id);
    return out;
}

Communicator::Communicator(const UniqueId& id, int rank, int world, int device) : rank_(rank), world_(world) {
    PORTTEN_CHECK(world >= 1 && rank >= 0 && rank < world, "dp: bad rank / world size");
    throw_if_error(pt_b200_set_device(device));
    ncclUniqueId nid;
    std::memcpy(&nid, id.data(), sizeof nid);
    ncclComm_t c = nullptr;
    nccl_check(ncclCommInitRank(&c, world, nid, rank), "ncclCommInitRank");
    comm_ = c;
}

Communicator::~Communicator() {
    if (comm_) ncclCommDestroy(as_comm(comm_));
}

void Communicator::allreduceGradients(DeviceTensor& gw, DeviceTensor* gb, void* stream) {
    PORTTEN_CHECK(gw.defined() && gw.isContiguous(), "dp: gradWeight must be a contiguous device tensor");
    PORTTEN_CHECK(!gb || (gb->defined() && gb->isContiguous()), "dp: gradBias must be a contiguous device tensor");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // one group: NCCL fuses both reductions into one launch on `stream`
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    nccl_check(ncclAllReduce(gw.data(), gw.data(), (size_t)gw.numel(), ncclFloat32, ncclSum, as_comm(comm_), st),
               "ncclAllReduce(gradWeight)");
    if (gb)
        nccl_check(ncclAllReduce(gb->data(), gb->data(), (size_t)gb->numel(), ncclFloat32, ncclSum, as_comm(comm_), st),
                   "ncclAllReduce(gradBias)");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

void Communicator::synchronize(void* stream, double timeout_s) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const int q = pt_b200_stream_query(stream);
        if (q == PT_OK) return;
        if (q != 1) {
            ncclCommAbort(as_comm(comm_));
            comm_ = nullptr;
            throw_if_error(q);
        }
        ncclResult_t async = ncclSuccess;
        nccl_check(ncclCommGetAsyncError(as_comm(comm_), &async), "ncclCommGetAsyncError");
        if (async != ncclSuccess && async != ncclInProgress) {
            ncclCommAbort(as_comm(comm_));
            comm_ = nullptr;
            throw BackendError(std::string("nccl: asynchronous error: ") + ncclGetErrorString(async));
        }
        const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (waited > timeout_s) {
            ncclCommAbort(as_comm(comm_));
            comm_ = nullptr;
            throw BackendError("nccl: collective did not complete within " + std::to_string(timeout_s) + " s");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

}  // namespace portten::dp
