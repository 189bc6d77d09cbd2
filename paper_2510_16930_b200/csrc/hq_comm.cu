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
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <memory>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

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

// ---------------------------------------------------------------- host transport
// Segment layout: a control block, then per rank an input slot and an output
// slot of `cap` doubles.  The whole segment is registered with CUDA
// (cudaHostRegister), so the D2H / H2D copies are DMA transfers that a stream
// capture records as memcpy nodes.
struct ShmCtrl {
    std::atomic<uint64_t> arrived;  // barrier: arrivals (monotone)
    std::atomic<uint32_t> attached;
    uint32_t world;
    uint64_t cap;
};

struct HostOp {  // one collective's host step, owned by the communicator
    HostXfer* x;
    int kind;     // 0 sum, 1 max, 2 row gather
    size_t count;
    std::vector<uint64_t> bounds;
    size_t row_elems;
};

struct HostXfer {
    int world = 1, rank = 0;
    std::string name;
    size_t bytes = 0;
    char* base = nullptr;
    ShmCtrl* ctrl = nullptr;
    double* slots = nullptr;  // [world][cap] inputs, then [world][cap] outputs
    uint64_t cap = 0;
    uint64_t phase = 0;       // barriers this rank passed
    std::vector<std::unique_ptr<HostOp>> ops;  // kept alive for the captured graphs
    double* in(int r) const { return slots + (size_t)r * cap; }
    double* out(int r) const { return slots + (size_t)(world + r) * cap; }

    void barrier() {
        ++phase;
        ctrl->arrived.fetch_add(1, std::memory_order_acq_rel);
        const uint64_t target = phase * (uint64_t)world;
        auto t0 = std::chrono::steady_clock::now();
        static const long limit_s = [] {  // HQ_HOST_BARRIER_S: give up (abort) after this many seconds
            const char* e = std::getenv("HQ_HOST_BARRIER_S");
            return e && std::atol(e) > 0 ? std::atol(e) : 300L;
        }();
        int spins = 0;
        while (ctrl->arrived.load(std::memory_order_acquire) < target) {
            if (++spins > 64) {
                sched_yield();
                spins = 0;
                if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(limit_s)) {
                    std::fprintf(stderr, "[hq] host transport %s: rank %d waited %ld s at barrier %llu; aborting\n",
                                 name.c_str(), rank, limit_s, (unsigned long long)phase);
                    std::abort();
                }
            }
        }
    }
};

// the host node: every rank's input slot is complete once all ranks pass the barrier; combine in rank order
// (the same bits on every rank), then a second barrier before any rank may overwrite its slot again
void CUDART_CB host_collective(void* p) {
    HostOp* op = static_cast<HostOp*>(p);
    HostXfer* x = op->x;
    x->barrier();
    double* o = x->out(x->rank);
    if (op->kind == 2) {
        for (int r = 0; r < x->world; ++r) {
            const size_t off = op->bounds[r] * op->row_elems, cnt = (op->bounds[r + 1] - op->bounds[r]) * op->row_elems;
            std::memcpy(o + off, x->in(r), cnt * sizeof(double));
        }
    } else {
        std::memcpy(o, x->in(0), op->count * sizeof(double));
        for (int r = 1; r < x->world; ++r) {
            const double* v = x->in(r);
            if (op->kind == 0)
                for (size_t i = 0; i < op->count; ++i) o[i] += v[i];
            else
                for (size_t i = 0; i < op->count; ++i) o[i] = o[i] >= v[i] ? o[i] : v[i];
        }
    }
    x->barrier();
}

void host_launch(const Comm& c, int kind, double* buf, size_t count, const uint64_t* bounds, size_t row_elems,
                 cudaStream_t s) {
    HostXfer* x = c.host;
    auto op = std::make_unique<HostOp>();
    op->x = x;
    op->kind = kind;
    op->count = count;
    op->row_elems = row_elems;
    size_t total = count;
    const double* src = buf;
    size_t send = count;
    if (kind == 2) {
        op->bounds.assign(bounds, bounds + c.world + 1);
        total = bounds[c.world] * row_elems;
        src = buf + bounds[c.rank] * row_elems;
        send = (bounds[c.rank + 1] - bounds[c.rank]) * row_elems;
    }
    if (total > x->cap) fail(HQ_ERR_CAPACITY, "host transport: collective of " + std::to_string(total) +
                                                  " doubles exceeds the segment's capacity " + std::to_string(x->cap));
    if (send) HQ_CUDA(cudaMemcpyAsync(x->in(c.rank), src, send * sizeof(double), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaLaunchHostFunc(s, host_collective, op.get()));
    if (total) HQ_CUDA(cudaMemcpyAsync(buf, x->out(c.rank), total * sizeof(double), cudaMemcpyHostToDevice, s));
    x->ops.push_back(std::move(op));
}

Comm::~Comm() {
    if (comm) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    if (host) {
        cudaStreamSynchronize(0);
        cudaHostUnregister(host->base);
        const uint32_t left = host->ctrl->attached.fetch_sub(1) - 1;
        munmap(host->base, host->bytes);
        if (left == 0) shm_unlink(host->name.c_str());
        delete host;
    }
}

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t s) const {
    if (!count) return;
    if (host) return host_launch(*this, 0, buf, count, nullptr, 0, s);
    if (!comm) return;  // one rank without NCCL: identity
    HQ_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s));
}

void Comm::allreduce_max(double* buf, size_t count, cudaStream_t s) const {
    if (!count) return;
    if (host) return host_launch(*this, 1, buf, count, nullptr, 0, s);
    if (!comm) return;
    HQ_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm), s));
}

void Comm::allgather_rows(double* buf, const uint64_t* bounds, size_t row_elems, cudaStream_t s) const {
    if (host) return host_launch(*this, 2, buf, 0, bounds, row_elems, s);
    if (!comm) return;
    HQ_NCCL(nccl().GroupStart());
    for (int r = 0; r < world; ++r) {
        const size_t off = bounds[r] * row_elems, cnt = (bounds[r + 1] - bounds[r]) * row_elems;
        if (cnt) HQ_NCCL(nccl().Broadcast(buf + off, buf + off, cnt, ncclFloat64, r, static_cast<ncclComm_t>(comm), s));
    }
    HQ_NCCL(nccl().GroupEnd());
}

void Comm::barrier(cudaStream_t s) const {
    if (world <= 1 || (!host && !comm)) return;
    if (!bar.p) {
        bar.alloc(1);
        HQ_CUDA(cudaMemsetAsync(bar.get(), 0, sizeof(double), s));
    }
    allreduce_sum(bar.get(), 1, s);
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

void require_unsharded(const DeviceTensor& T, const char* what) {
    if (T.shard_world > 1)
        fail(HQ_ERR_SHAPE, std::string(what) + ": the tensor keeps only this rank's rows (hq_tensor_shard); "
                                               "use it with a distributed solver of the same partition");
}

namespace {
template <typename T>
void keep_slice(DBuf<T>& b, uint64_t z0, uint64_t z1, size_t pad, cudaStream_t s) {
    if (!b.p) return;
    // the pass kernels stage contiguous record slices with 16-byte copies from the 16-byte-aligned global
    // position at or below the slice start: keep the slice from such a position so get() + z keeps the
    // alignment of the unsharded stream for every z
    z0 -= z0 % (16 / sizeof(T) ? 16 / sizeof(T) : 1);
    DBuf<T> nb;
    nb.alloc(z1 - z0 + pad);
    HQ_CUDA(cudaMemcpyAsync(nb.p, b.get() + z0, sizeof(T) * (z1 - z0 + pad), cudaMemcpyDeviceToDevice, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    nb.off = z0;
    b = std::move(nb);
}
}  // namespace

void shard_tensor(DeviceTensor& T, int world, int rank, cudaStream_t s) {
    if (world < 1 || rank < 0 || rank >= world) fail(HQ_ERR_SHAPE, "invalid world size / rank");
    if (T.shard_world > 1) fail(HQ_ERR_SHAPE, "tensor is already sharded");
    if (world == 1) return;
    for (int n = 0; n < T.order; ++n) {
        ModeLayout& L = T.modes[n];
        std::vector<int64_t> off(L.rows + 1);
        HQ_CUDA(cudaMemcpyAsync(off.data(), L.rowptr.get(), sizeof(int64_t) * off.size(), cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        std::vector<uint64_t> uo(off.begin(), off.end());
        std::vector<uint64_t> bnd(world + 1);
        partition_rows(uo.data(), L.rows, world, bnd.data());
        const uint64_t z0 = uo[bnd[rank]], z1 = uo[bnd[rank + 1]];
        // the streams carry tail padding the pass kernels' 16-byte staging reads into (hq_layout.cu)
        const size_t padv = L.val.n - T.nnz, padi = (T.order > 1 && L.idx[0].p) ? L.idx[0].n - T.nnz : 0;
        keep_slice(L.val, z0, z1, padv, s);
        for (int q = 0; q < T.order - 1; ++q) keep_slice(L.idx[q], z0, z1, padi, s);
        L.entries.release();
        T.shard_bounds[n] = bnd;
    }
    T.coords.release();
    T.vals.release();
    T.shard_world = world;
    T.shard_rank = rank;
}

Comm* comm_create_host(int world, int rank, const char* name, uint64_t cap) {
    if (world < 1 || rank < 0 || rank >= world) fail(HQ_ERR_SHAPE, "invalid world size / rank");
    if (!name || name[0] != '/') fail(HQ_ERR_SHAPE, "host transport: segment name must start with '/'");
    const size_t bytes = 4096 + (size_t)2 * world * cap * sizeof(double);
    int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) fail(HQ_ERR_CUDA, std::string("host transport: shm_open failed for ") + name);
    if (ftruncate(fd, (off_t)bytes) != 0) {
        close(fd);
        fail(HQ_ERR_CUDA, "host transport: ftruncate failed");
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) fail(HQ_ERR_CUDA, "host transport: mmap failed");
    auto* x = new HostXfer();
    x->world = world;
    x->rank = rank;
    x->name = name;
    x->bytes = bytes;
    x->base = static_cast<char*>(p);
    x->ctrl = reinterpret_cast<ShmCtrl*>(x->base);  // zero-filled by ftruncate on creation
    x->slots = reinterpret_cast<double*>(x->base + 4096);
    x->cap = cap;
    x->ctrl->attached.fetch_add(1);
    cudaError_t e = cudaHostRegister(x->base, bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        munmap(x->base, bytes);
        delete x;
        fail(HQ_ERR_CUDA, std::string("host transport: cudaHostRegister: ") + cudaGetErrorString(e));
    }
    auto* c = new Comm();
    c->world = world;
    c->rank = rank;
    c->host = x;
    x->barrier();  // every rank attached before the first collective
    return c;
}

}  // namespace hq
