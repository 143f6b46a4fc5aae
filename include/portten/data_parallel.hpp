// Batch-sharded data parallelism for the conv layers in the C++ operator API (
// the Python twin is paper_1606_04884_b200/dp.py). The reference has no multi-device path
// (SPEC.md:325-326 lists it as a non-goal); this is new work.
//
// The minibatch is the only sharded dimension: updateOutput / updateGradInput are per-image
// independent, so the one exchange is a sum-allreduce of each layer's gradWeight and
// gradBias. It runs over NCCL (NVLink / NVSwitch on a B200 node) on the caller's stream —
// gradWeight and gradBias in one NCCL group, i.e. one fused launch — so a CUDA graph or a
// communication stream can order it against the next layer's kernels. synchronize() polls
// ncclCommGetAsyncError while it waits, so a failed or hung peer surfaces as a BackendError
// (and the communicator is aborted) instead of a silent hang.
#pragma once

#include <array>
#include <cstdint>

#include "portten/tensor.hpp"

namespace portten::dp {

struct ShardRange {
    std::int64_t start, stop;  // [start, stop) of the global batch this rank owns
};
/// Images of rank `rank` out of `world`; the remainder goes to the low ranks
/// (identical to dp.shard_range in the Python package).
ShardRange shard_range(std::int64_t n, int rank, int world);

/// NCCL's unique id (ncclUniqueId, 128 bytes). Rank 0 creates it and the caller distributes
/// it to the other ranks (a file, MPI, a TCP store ...).
using UniqueId = std::array<char, 128>;
UniqueId new_unique_id();

class Communicator {
public:
    /// One rank per GPU: binds `device` and joins the `world`-rank communicator of `id`.
    Communicator(const UniqueId& id, int rank, int world, int device);
    ~Communicator();
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;

    int rank() const { return rank_; }
    int world() const { return world_; }

    /// gw (and gb when non-null) <- sum over ranks, in place, enqueued on `stream`.
    /// Both tensors must be contiguous device tensors.
    void allreduceGradients(DeviceTensor& gw, DeviceTensor* gb, void* stream);

    /// Wait until `stream` has drained, polling the communicator's asynchronous error state;
    /// throws BackendError (after aborting the communicator) on an NCCL error or timeout.
    void synchronize(void* stream, double timeout_s = 600.0);

private:
    void* comm_ = nullptr;  // ncclComm_t
    int rank_ = 0, world_ = 1;
};

}  // namespace portten::dp
