// hq_dense.cuh — tall-skinny orthogonalisation and the K x K steps.
#pragma once

#include <memory>

#include "hq_plan.cuh"

namespace hq {

constexpr int kMaxRank = 32;
constexpr int kAcc = (kMaxRank * kMaxRank + 255) / 256;  // K*K entries per thread (256 threads)

// CholeskyQR2 of A (rows x K) with fused side products, all on the device.
// Scratch owned by the caller (sizes from dense_scratch_doubles()).
struct QrScratch {
    double* wpart;   // [dense slots][K*K]
    double* w;       // K*K
    double* r1inv;   // K*K
    double* rinv;    // K*K
    double* ppart;   // [dense slots][K*K]
    double* maxv;    // 1
    double* hh;      // Householder workspace: rows*K + rows (reflectors) + K
};

int dense_slots();

// X = A T (T null: identity); out <- X (optional); part[cta] = X^T Y with
// Y = other (optional) or X; maxpart[cta] = max|A| (optional).  hq_rowgemm.cu
bool rowgemm_supported(int K);
constexpr int kMaxPeers = 15;  // other ranks of one node
struct RowGemm {
    const double* A;       // rows x K
    uint64_t rows;
    const double* T;       // first transform (null: identity)
    const double* T2;      // optional second transform: X = fl(fl(A T) T2) (the first stage never leaves the SM)
    const double* alt;     // optional: when st->shifted, X = alt T2 instead (one stage; the shifted apply)
    double* out;           // X (optional; may alias A / alt)
    const double* other;   // part = X^T other (optional; else the Gram X^T X)
    double* part;          // [CTA][K*K] partials
    double* maxpart;       // [CTA] max|A| (optional)
    const DevStatus* st;
    int run_if;
    // multi-GPU: the same rows of X also stored straight into the other ranks' replicas of the factor (peer
    // memory mapped through CUDA IPC: NVLink / NVSwitch stores) -- the apply and the all-gather of U_new in one
    // kernel, the transfer overlapping the row products chunk by chunk.  Pointers are to the same row as `out`.
    double* peer_out[kMaxPeers];
    int npeer;
};
void launch_rowgemm(int K, const RowGemm& g, cudaStream_t s);
void launch_rowgemm(int K, const double* A, uint64_t rows, const double* T, double* out, const double* other,
                    double* part, double* maxpart, const DevStatus* st, int run_if, cudaStream_t s);

// W = sum of `nslots` partial K*K slots (fixed order) and max over max partials
void launch_reduce_pass(const double* mpart, int mlen, const double* wpart, int wlen, const double* maxpart,
                        int nslots, double* m_out, double* w_out, double* max_out, const DevStatus* st, int run_if,
                        cudaStream_t s);
// W = A^T A and max|A| for a standalone QR
void launch_gram(const double* A, uint64_t rows, int K, double* wpart, double* maxpart, const DevStatus* st,
                 int run_if, cudaStream_t s);
// degeneracy test (max|A| == 0 -> abort with the 1-based mode when
// degenerate_mode > 0), Cholesky of W, inverse of R1; sets st->fallback when
// CholeskyQR2 would lose accuracy
void launch_chol1(const double* w, const double* maxv, int K, double* r1inv, DevStatus* st, int degenerate_mode,
                  uint64_t m_rows, cudaStream_t s, bool abort_on_fallback = false);
// the partials of W2 = Q1^T Q1, Q1 = A R1^-1 (not written: recomputed bit for bit by gram3 / apply_qr)
void launch_gram2(const double* A, uint64_t rows, int K, const double* r1inv, double* wpart, const DevStatus* st,
                  cudaStream_t s);
// Cholesky of W2 (reduced from partials): rinv = R2^-1, rc = R1^-1 R2^-1; if
// m != null and the update is not shifted, G_(n) = rc^T M refolded into the
// core layout (core_out)
// multi-GPU: abort 3 cleared, fallback armed for the host-driven Householder continuation
void launch_dist_resume(DevStatus* st, cudaStream_t s);
void launch_chol2(const double* wpart, int nslots, int K, const double* r1inv, double* rinv, double* rc,
                  const double* m, const ModeShape* sh, double* core_out, DevStatus* st, cudaStream_t s,
                  bool abort_on_fallback = false, int mode1 = 0);
// shifted CholeskyQR3 third pass (RunIf kOnlyShifted): Q2 = (A R1^-1) R2^-1
// written to q_out and the partials of W3 = Q2^T Q2; then rinv = R3^-1 with the
// identity and rank checks (rc = R1^-1 R2^-1 for diag R, wfull = A^T A for ||A||_F)
void launch_gram3(const double* A, uint64_t rows, int K, const double* r1inv, const double* r2inv, double* q_out,
                  double* wpart, const DevStatus* st, cudaStream_t s);
void launch_chol3(const double* wpart, int nslots, int K, const double* rc, double* rinv, const double* wfull,
                  DevStatus* st, cudaStream_t s, bool abort_on_fallback = false);
// U = A Rinv (written to u_out when non-null, which may alias A); P partials
// of U^T U_old when u_old non-null.  apply=false: U read from u_out (fallback
// drift).
void launch_apply(const double* A, uint64_t rows, int K, const double* rinv, double* u_out, const double* u_old,
                  double* ppart, bool apply, const DevStatus* st, int run_if, cudaStream_t s);
// the CholeskyQR product U = (A R1^-1) R2^-1 (two stages, each rounded as if materialised) written to
// u_out, and the partials of P = U^T U_old (u_old optional).  shifted_alt: when st->shifted, U = u_out R3^-1
// instead (u_out holds Q2 from gram3, rinv holds R3^-1 from chol3)
void launch_apply_qr(const double* A, uint64_t rows, int K, const double* r1inv, const double* rinv, double* u_out,
                     const double* u_old, double* ppart, bool shifted_alt, const DevStatus* st, int run_if,
                     cudaStream_t s,
                     double* const* peer_out = nullptr, int npeer = 0);
// drift = max(2K - 2 ||P||_*, 0) (manifold.cpp:55-60) from P partials; when
// `objective` non-null also f = ||G||^2 and fit = dns - f for the sweep;
// `end_of_sweep` advances the sweep counter and applies the stop rule.
struct SweepTrace {
    double* objective;   // [max_sweeps]
    double* fit;         // [max_sweeps]
    double* drift;       // [max_sweeps * order]
    double* fit_prev;    // 1
    const double* grad;  // [max_sweeps * order] per-update grad_norm_sq, or null (no gradient stop)
    int order;
    double tol_grad;     // solvers.cpp:165-167 stop when > 0
    unsigned long long* t_end;  // [max_sweeps] device timestamp (ns) at the end of each sweep, or null
};

// Per-update gradient diagnostics (ModeUpdateRecord, solvers.hpp:40-49)
struct UpdTrace {
    double* grad;        // [max_sweeps * order]
    double* f_before;    // [max_sweeps * order]
    double* sigma;       // [max_sweeps * order * kstride]
    double* lambda;      // [max_sweeps * order * kstride]
    unsigned long long* t;  // [max_sweeps * order] device timestamp (ns) of the diagnostics point
    int kstride;
};
// pre-update diagnostics of mode `mode` (solvers.cpp:126-137; manifold.cpp:37-84):
// W = A^T A (reduced), gt = G_(n)^T (L x K).  Raises abort 5 (DiagnosticError)
// or 6 (ContractError) like the reference.
void launch_update_diag(const double* w, const double* gt, int K, int L, int mode, int order, const UpdTrace& tr,
                        DevStatus* st, cudaStream_t s);
void launch_drift(const double* ppart, int nslots, int K, const double* core, uint64_t core_size, double dns,
                  int order, int mode, bool end_of_sweep, double tol, uint64_t max_sweeps, const SweepTrace& tr,
                  DevStatus* st, cudaStream_t s);
// P (reduced) -> trace slot of the current sweep (trp[sweep][mode][kmax^2])
void launch_store_p(const double* ppart, int nslots, int K, int order, int mode, int kmax, uint64_t max_sweeps,
                    double* trp, const DevStatus* st, cudaStream_t s);
// objective / fit / stop rule at the end of a sweep
void launch_sweep_end(const double* core, uint64_t core_size, double dns, double tol, uint64_t max_sweeps,
                      const SweepTrace& tr, DevStatus* st, cudaStream_t s);
// drifts of `pairs` (sweep, mode) trace slots; ranks: device array of the N ranks
void launch_drift_batch(const double* trp, int pairs, int order, const int* ranks_dev, int kmax, double* drift,
                        cudaStream_t s);
// Householder QR following dense_core.cpp:127-198 step for step, one CTA per
// SM with grid barriers (cooperative launch).  The rank-deficiency fill
// (rng.hpp:13-35, seed 0x48514F5251) reads the precomputed normal stream
// `table` (table_len normals; see fill_table) and falls back to drawing on the
// device when the table is absent or too short.  work: householder_work_doubles
// doubles (any rows x K up to the size it was made for), its control block
// zeroed once by householder_reset (barrier counters reset themselves).
size_t householder_work_doubles(uint64_t rows, int K);
void householder_reset(double* work, cudaStream_t s);
void launch_householder(const double* A, uint64_t rows, int K, double* q_out, double* work, const double* table,
                        uint64_t table_len, const DevStatus* st, int run_if, cudaStream_t s);
// the fill stream: the first `count` normals of tucker::Rng(0x48514F5251)
// (rng.hpp:13-35), generated on the host once per process (per device) and
// kept on the device; a holder keeps its table alive (graphs capture the
// pointer).  Null when count exceeds kFillTableCap.
struct FillTable {
    DBuf<double> buf;
    uint64_t len = 0;
};
constexpr uint64_t kFillTableCap = 1ull << 28;
std::shared_ptr<const FillTable> fill_table(uint64_t count);

// tucker::Rng helpers on the host (rng.hpp): mix_seed, and `count` normals of
// Rng(seed) (raw draws sequential, Box-Muller threaded)
uint64_t mix_seed(uint64_t seed, uint64_t salt);
void gaussian_stream(uint64_t seed, uint64_t count, double* out);

// qr_orthonormal on the device (dense_core.cpp:127-198): CholeskyQR2 /
// shifted CholeskyQR3 / multi-CTA Householder (with the reference's fill)
struct QrWork {
    DBuf<double> wpart, maxpart, w, maxv, r1inv, rinv, rc, ppart, hh;
    DBuf<DevStatus> st;
    void ensure(uint64_t rows, int K);
};
void qr_device(const double* A, uint64_t rows, int K, double* Q, QrWork& w, cudaStream_t s);
void check_rank_limits(int K);
// G_(n)^T (L x K_n) from the core
void launch_gt(const double* core, const ModeShape& sh, const int* ranks, double* gt, const DevStatus* st,
               cudaStream_t s);
// core_out = reduce of M partials (mode 0 unfolding == core layout)
void launch_reduce_core(const double* mpart, int nslots, uint64_t size, double* core_out, const DevStatus* st,
                        int run_if, cudaStream_t s);
// core = reduce of the M partials of a kCore pass over mode sh.n, refolded into the core layout
void launch_reduce_core_mode(const double* mpart, int nslots, const ModeShape& sh, double* core_out,
                             const DevStatus* st, int run_if, cudaStream_t s);
// ||G||^2 into *out (deterministic)
void launch_core_normsq(const double* core, uint64_t size, double* out, cudaStream_t s);
// max_ij |U^T U - I| over all modes' final factors
void launch_defect(const double* u, uint64_t rows, int K, double* wpart, double* out_max, cudaStream_t s);

}  // namespace hq
