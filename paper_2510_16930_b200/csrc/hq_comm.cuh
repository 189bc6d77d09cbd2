// hq_comm.cuh — communicator and row partition planner (hq_comm.cu).
#pragma once

#include "hq_internal.cuh"

namespace hq {

// Contiguous whole-row ranges with ~nnz/world nonzeros each:
// rank r owns rows [bounds[r], bounds[r+1]).  Host-only (CPU-testable).
void partition_rows(const uint64_t* offsets, uint64_t rows, int world, uint64_t* bounds);

struct HostXfer;  // host transport state (hq_comm.cu)

// Collectives of the distributed solve, on the solver's stream (capturable).
// Two transports: NCCL (one process per GPU; NVLink / NVSwitch) and a host
// transport for ranks that share a node but not a GPU fabric -- ranks exchange
// through a POSIX shared-memory segment: a D2H copy into the rank's slot, a
// host node that waits for every rank and combines the slots in rank order,
// and an H2D copy of the result.  No kernel ever waits on another rank, so the
// host transport is safe with several ranks on one GPU (what the multi-rank
// GPU test uses: gpurun provides one GPU).
struct Comm {
    int world = 1;
    int rank = 0;
    void* comm = nullptr;     // ncclComm_t
    HostXfer* host = nullptr;  // host transport
    ~Comm();
    void allreduce_sum(double* buf, size_t count, cudaStream_t s) const;
    void allreduce_max(double* buf, size_t count, cudaStream_t s) const;
    // every rank's rows [bounds[r], bounds[r+1]) of a row-major buffer, broadcast from their owner
    void allgather_rows(double* buf, const uint64_t* bounds, size_t row_elems, cudaStream_t s) const;
    // every rank's work enqueued on its stream before this point is complete before any rank's work after it
    // starts (an 8-byte all-reduce): orders the peer-memory stores of the fused apply against their readers
    void barrier(cudaStream_t s) const;
    mutable DBuf<double> bar;  // the barrier's operand
};

void nccl_unique_id(uint8_t* out128);
// Row-partitioned storage for a distributed solve: per mode, keep only the stream slice (values + index
// streams) of this rank's rows -- the same partition the solver uses (partition_rows over the mode's
// offsets) -- and free the lexicographic copy and the buckets' entries.  Kernels keep indexing streams
// with global positions (DBuf::off).
void shard_tensor(DeviceTensor& T, int world, int rank, cudaStream_t s);
void require_unsharded(const DeviceTensor& T, const char* what);
Comm* comm_create(int world, int rank, const uint8_t* id128);
// host transport over the shared-memory segment `name` (created by whichever rank comes first); `cap` is the
// largest collective in doubles (a factor: max I_n K_n)
Comm* comm_create_host(int world, int rank, const char* name, uint64_t cap);

}  // namespace hq

struct hq_comm {
    hq::Comm* impl = nullptr;
    ~hq_comm() { delete impl; }
};
