// hq_comm.cuh — communicator and row partition planner (hq_comm.cu).
#pragma once

#include "hq_internal.cuh"

namespace hq {

// Contiguous whole-row ranges with ~nnz/world nonzeros each:
// rank r owns rows [bounds[r], bounds[r+1]).  Host-only (CPU-testable).
void partition_rows(const uint64_t* offsets, uint64_t rows, int world, uint64_t* bounds);

struct Comm {
    int world = 1;
    int rank = 0;
    void* comm = nullptr;  // ncclComm_t
    ~Comm();
    void allreduce_sum(double* buf, size_t count, cudaStream_t s) const;
    void allreduce_max(double* buf, size_t count, cudaStream_t s) const;
    // every rank's rows [bounds[r], bounds[r+1]) of a row-major buffer, broadcast from their owner
    void allgather_rows(double* buf, const uint64_t* bounds, size_t row_elems, cudaStream_t s) const;
};

void nccl_unique_id(uint8_t* out128);
Comm* comm_create(int world, int rank, const uint8_t* id128);

}  // namespace hq

struct hq_comm {
    hq::Comm* impl = nullptr;
    ~hq_comm() { delete impl; }
};
