// hq_plan.cuh — work decomposition of a mode-sorted stream and the sparse
// pass entry points (hq_pass.cu).
#pragma once

#include "hq_internal.cuh"

namespace hq {

// Rows with more nonzeros than kShortMax are "long": they are cut into
// segments of at most kSegLen nonzeros, each reduced by one CTA into a
// partial Kronecker row, and the partials of a row are summed in segment
// order (deterministic).  All other rows are processed whole by the tile
// kernels.
#ifndef HQ_SHORT_MAX
#define HQ_SHORT_MAX 256
#endif
constexpr int64_t kShortMax = HQ_SHORT_MAX;
constexpr int64_t kSegLen = 4096;
// long-row threshold of a skewed order-3 mode whose long rows run through the fiber units (hq_pass.cu
// plan_mode; measured on config 3: 256 -> 7.8, 128 -> 7.3, 64 -> 7.2, 48 -> 7.1, 32 -> 7.2, 16 -> 7.8 ms / sweep)
constexpr int64_t kSkewedShortMax = 64;

void plan_mode(ModeLayout& L, uint64_t nnz, int order, cudaStream_t s);

double device_sum_sq(const double* v, uint64_t n, cudaStream_t s);
// vals_ready (optional): the values are still arriving (an H2D copy on another stream that records this
// event); the coordinate-only work (range checks, key packing, lexicographic sort) runs before s waits on it
void build_tensor(DeviceTensor& T, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords_dev,
                  const double* vals_dev, cudaStream_t s, cudaEvent_t vals_ready = nullptr);
void export_buckets(const DeviceTensor& T, int mode, uint64_t* offsets, uint64_t* entries, cudaStream_t s);
}  // namespace hq
struct hq_tns;
namespace hq {
// `.tns` text -> COO (hq_tns.cu); throws hq::Error like the reference's load_tns
void tns_parse(const char* text, uint64_t len, int ovr_order, const uint64_t* ovr_dims, hq_tns& out);

// Device status word shared by every kernel of a solve.  Kernels return early
// when `abort` is set; the CholeskyQR kernels run only while `fallback` is 0,
// the Householder fallback kernels only while it is 1.  `shifted` marks a
// mode update whose Gram matrix was too ill-conditioned for plain CholeskyQR2:
// it runs shifted CholeskyQR3 (a third Gram pass) and recomputes the core with
// a sparse pass instead of R^-T M.
struct DevStatus {
    int abort;
    int degenerate_mode;   // 1-based mode of the first A == 0 (solvers.cpp:124)
    int degenerate_sweep;
    int fallback;          // current QR needs the Householder path
    unsigned int fallback_count;
    int sweep;             // 1-based sweep counter (advanced on the device)
    int shifted;           // current QR runs shifted CholeskyQR3
    unsigned int shifted_count;
    int diag_code;         // abort 5/6 detail: 1 negative gradient, 2 interlacing, 3 not PSD
    int diag_k;            // 1-based index for interlacing
    unsigned int dist_hh_count;    // multi-GPU: updates finished by the host-driven Householder continuation
    int pending_mode;              // multi-GPU, abort 3: 1-based mode whose update needs that continuation
};

enum RunIf { kAlways = 0, kOnlyFallback = 1, kOnlyCholQR = 2, kOnlyShifted = 3, kFallbackOrShifted = 4 };

__device__ __forceinline__ bool skip_kernel(const DevStatus* st, int run_if) {
    if (!st) return false;
    if (st->abort) return true;
    if (run_if == kOnlyFallback) return st->fallback == 0;
    if (run_if == kOnlyCholQR) return st->fallback != 0;
    if (run_if == kOnlyShifted) return st->fallback != 0 || st->shifted == 0;
    if (run_if == kFallbackOrShifted) return st->fallback == 0 && st->shifted == 0;
    return false;
}

// What a sparse pass computes per row i (Y_i = the Kronecker row of mode n):
//   kTTMcTC: a_i = Y_i G_(n)^T                 (kernels.cpp:86-163 output row)
//   kCore:   a_i = U_n[i, :]                   (so M = sum a_i^T Y_i = G_(n), kernels.cpp:40-84)
// and always accumulates M = sum_i a_i^T Y_i (K_n x L), W = sum a_i^T a_i
// (K_n x K_n) and max |a| into per-CTA partial slots.
// kTTMcTCOnly: the standalone TTMcTC call (kernels.cpp:86-163) -- A only; the short-row fast kernels skip
// the M / W accumulation (other kernels run it as kTTMcTC and the partials are ignored)
enum PassKind { kTTMcTC = 0, kCore = 1, kTTMcTCOnly = 2 };

// G_(n)^T buffers (k_gt) carry, after the L x K_n matrix, the K = 10 order-3 short-row pass's pre-permuted
// A-GEMM fragments (hq_dense.cu k_gt, hq_pass_fast.cu k_pass_np3): allocate gt_doubles(sh)
constexpr int kGtFragTable = 25 * 32 + 25 * 8;
__host__ __device__ inline bool gt_frag_table(const ModeShape& sh) {
    return sh.order == 3 && sh.ko[0] == 10 && sh.ko[1] == 10 && sh.kn == 10;
}
inline size_t gt_doubles(const ModeShape& sh) { return (size_t)sh.L * sh.kn + (gt_frag_table(sh) ? kGtFragTable : 0); }

struct PassOut {
    double* A;        // I_n x K_n rows (may be null for kCore)
    double* mpart;    // [slots][K_n * L]
    double* wpart;    // [slots][K_n * K_n]
    double* maxpart;  // [slots]
    double* ypart;    // [long_segments][L] scratch
};

// Number of partial slots a pass over this mode uses.
int pass_slots(const ModeLayout& L, const ModeShape& sh);
size_t pass_ypart_doubles(const ModeLayout& L, const ModeShape& sh);

// Launches the pass kernels (no host synchronisation; graph-capturable).
// gt = G_(n)^T as L x K_n (kTTMcTC only).
// Only rows [row_begin, row_end) of the mode-n unfolding are processed (the
// rank's share in a multi-GPU solve; the whole mode by default).
void launch_pass(const DeviceTensor& T, int mode, const ModeShape& sh, const FactorPtrs& f, PassKind kind,
                 const double* gt, const PassOut& out, const DevStatus* st, int run_if, cudaStream_t s,
                 uint64_t row_begin = 0, uint64_t row_end = ~0ull);
// number of kernels launch_pass issues
int pass_launch_count(const ModeLayout& L, const ModeShape& sh);

}  // namespace hq
