// hq_comm.cu — multi-GPU plumbing: NCCL (loaded at run time), the row
// partition planner, and the communicator object of the C-ABI.
//
// One process per GPU.  Every rank builds the same tensor layout; for each
// mode the rows of the mode-n unfolding are split into contiguous ranges with
// ~nnz/P nonzeros each (whole rows, so each rank owns the A / U rows it
// writes — the parallelism contract of SPEC.md:247).  Factors and the core
// are replicated.  Per mode update the K x K / K x L partial sums are
// all-reduced and the new factor rows are broadcast from their owners
// (grouped broadcasts = a variable-block all-gather), all on the solver's
// stream, so the sweep graph captures them.
//
// libnccl.so.2 is dlopen'ed on first use: single-GPU users never need it, and
// inside a PyTorch process the already-loaded NCCL is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "hq_comm.cuh"

namespace hq {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Broadcast &&
                 api.GroupStart && api.GroupEnd && api.GetErrorString;
    });
    if (!api.ok) fail(HQ_ERR_NCCL, "libnccl.so.2 not found or incomplete");
    return api;
}

#define HQ_NCCL(call)                                                                             \
    do {                                                                                          \
        ncclResult_t _r = (call);                                                                 \
        if (_r != ncclSuccess) ::hq::fail(HQ_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(_r)); \
    } while (0)

}  // namespace

void partition_rows(const uint64_t* offsets, uint64_t rows, int world, uint64_t* bounds) {
    // bounds[r] = first row of rank r: the smallest row i with offsets[i] >= r * nnz / world
    // (whole rows; empty ranks allowed when a single row outweighs a share)
    const uint64_t nnz = offsets[rows];
    bounds[0] = 0;
    for (int r = 1; r < world; ++r) {
        const uint64_t target = (uint64_t)((unsigned __int128)nnz * r / world);
        uint64_t lo = bounds[r - 1], hi = rows;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (offsets[mid] >= target) hi = mid; else lo = mid + 1;
        }
        bounds[r] = lo;
    }
    bounds[world] = rows;
}

Comm::~Comm() {
    if (comm) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
}

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t s) const {
    if (!comm || !count) return;  // one rank without NCCL: identity
    HQ_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s));
}

void Comm::allreduce_max(double* buf, size_t count, cudaStream_t s) const {
    if (!comm || !count) return;
    HQ_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm), s));
}

void Comm::allgather_rows(double* buf, const uint64_t* bounds, size_t row_elems, cudaStream_t s) const {
    if (!comm) return;
    HQ_NCCL(nccl().GroupStart());
    for (int r = 0; r < world; ++r) {
        const size_t off = bounds[r] * row_elems, cnt = (bounds[r + 1] - bounds[r]) * row_elems;
        if (cnt) HQ_NCCL(nccl().Broadcast(buf + off, buf + off, cnt, ncclFloat64, r, static_cast<ncclComm_t>(comm), s));
    }
    HQ_NCCL(nccl().GroupEnd());
}

void nccl_unique_id(uint8_t* out128) {
    ncclUniqueId id;
    HQ_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
}

Comm* comm_create(int world, int rank, const uint8_t* id128) {
    if (world < 1 || rank < 0 || rank >= world) fail(HQ_ERR_SHAPE, "invalid world size / rank");
    auto* c = new Comm();
    c->world = world;
    c->rank = rank;
    // a one-rank communicator needs no NCCL; HQ_NCCL_ONE_RANK=1 builds a real one-rank NCCL communicator
    // anyway (exercises the NCCL calls inside the captured sweep on one GPU)
    const char* force = std::getenv("HQ_NCCL_ONE_RANK");
    if (world > 1 || (force && force[0] == '1')) {
        ncclUniqueId id;
        std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t nc = nullptr;
        ncclResult_t r = nccl().CommInitRank(&nc, world, id, rank);
        if (r != ncclSuccess) {
            delete c;
            fail(HQ_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
        }
        c->comm = nc;
    }
    return c;
}

}  // namespace hq
