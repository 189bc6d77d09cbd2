/*
 * hoqri_b200.h — the C-ABI of the B200 HOQRI engine (libhoqri_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (arxiv 2510.16930, /root/reference/proj) is a C++ static library whose
 * callers link `tucker::` symbols directly; it has no FFI.  Every entry point
 * below replaces one reference function (cited as file:line, relative to
 * /root/reference/proj).  The C++ shim libtucker_b200.so
 * (paper_2510_16930_b200/csrc/tucker_shim.cpp) re-exposes the reference's
 * `tucker::` signatures on top of this ABI, and the Python mirror
 * (paper_2510_16930_b200/__init__.py) binds it with ctypes.
 *
 * Rules:
 *  - Plain pointers and sizes only.  Pointers are HOST pointers unless the
 *    name ends in `_dev`.  Sizes are uint64_t / int64_t.
 *  - No exception crosses this boundary.  Every call returns an hq_status;
 *    hq_last_error() holds a thread-local message and hq_last_error_payload()
 *    the 1-based mode of a DEGENERATE error (errors.hpp:73-80) or the line of
 *    a PARSE error (errors.hpp:17-22).
 *  - Matrices are row-major (dense_core.hpp:10-22); factor sets are passed as
 *    an array of N pointers, factor n of shape dims[n] x ranks[n]; the core is
 *    K_1 x ... x K_N with the last mode fastest (dense_core.hpp:33-43).
 *  - `stream` is a cudaStream_t passed as an opaque pointer (NULL = the
 *    library's default stream).  Calls that return host results synchronise
 *    that stream before returning.
 */
#ifndef HOQRI_B200_H
#define HOQRI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:9-70 taxonomy, plus device failures */
typedef enum hq_status {
    HQ_OK = 0,
    HQ_ERR_SHAPE = 1,       /* ShapeError */
    HQ_ERR_RANGE = 2,       /* RangeError */
    HQ_ERR_VALUE = 3,       /* ValueError */
    HQ_ERR_PARSE = 4,       /* ParseError (payload: line) */
    HQ_ERR_CAPACITY = 5,    /* CapacityError */
    HQ_ERR_CONTRACT = 6,    /* ContractError */
    HQ_ERR_DIAGNOSTIC = 7,  /* DiagnosticError */
    HQ_ERR_DEGENERATE = 8,  /* DegenerateStateError (payload: mode, 1-based) */
    HQ_ERR_INFEASIBLE = 9,  /* InfeasibleError */
    HQ_ERR_CUDA = 10,       /* CUDA runtime / kernel failure */
    HQ_ERR_NCCL = 11,       /* NCCL failure (multi-GPU) */
    HQ_ERR_INTERNAL = 12
} hq_status;

const char* hq_last_error(void);
int64_t hq_last_error_payload(void);
const char* hq_version(void);
/* Device buffers freed by tensors / solvers are kept on the engine's free lists for the next solve (no driver
   allocation in steady state; HQ_POOL_RELEASE_GB caps them).  This returns them to the driver; *freed_bytes (may be
   NULL) receives the amount.  Engine-only (the reference is a CPU library and has no counterpart). */
int hq_release_cached_memory(uint64_t* freed_bytes);

/* ---------------------------------------------------------------- tensor --
 * Device-resident mirror of tucker::SparseTensor.  Creation validates the
 * input (sparse_tensor.cpp:22-38: RANGE for a coordinate >= extent, VALUE for
 * a non-finite value, SHAPE for order 0 / zero extent / size mismatch), sorts
 * the entries lexicographically, merges duplicates by summing
 * (sparse_tensor.cpp:43-71), builds every mode's buckets
 * (sparse_tensor.cpp:73-89) and the mode-sorted streams the kernels read.
 * All of it runs on the device.  Replaces SparseTensor::SparseTensor
 * (sparse_tensor.hpp:37-38). */
typedef struct hq_tensor hq_tensor;

int hq_tensor_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                     const double* values, void* stream, hq_tensor** out);
/* same, but coords/values already in device memory (not modified) */
int hq_tensor_create_dev(int order, const uint64_t* dims, uint64_t nnz,
                         const uint32_t* coords_dev, const double* values_dev, void* stream,
                         hq_tensor** out);
int hq_tensor_destroy(hq_tensor* t);
/* order, nnz after merging (sparse_tensor.hpp:40-42) */
int hq_tensor_info(const hq_tensor* t, int* order, uint64_t* dims, uint64_t* nnz);
/* Work plan of one mode's unfolding (engine-side, no reference counterpart): rows, non-empty rows,
   long rows (> 256 nonzeros, segmented), their segments, and hot = 1 when the mode is skewed (rows longer
   than 32x the mean hold >= 5% of the nonzeros) so its factor is gathered L1-allocating by the other passes,
   and max_tile32 = the most short-row nonzeros in one 32-row tile of the pass kernels */
int hq_tensor_mode_plan(const hq_tensor* t, int mode, uint64_t* rows, uint64_t* nonempty_rows, uint64_t* long_rows,
                        uint64_t* long_segments, int* hot, uint64_t* max_tile32);
/* fiber units of a mode's long rows (order 3, skewed tensors; engine-only, no reference counterpart): within a
   row the nonzeros sharing the first other index form a fiber, whose Kronecker product is taken once
   (kernels.cpp:86-163 takes it per nonzero; same sum, regrouped).  units = 0 when the mode does not use them;
   long_nnz / units is the factor by which the long rows' stream shrinks; short_max = the mode's long-row
   threshold (256; 64 for a skewed mode that uses the units).  HQ_FIBERS=0/1 (read when the tensor is built)
   disables / forces them. */
int hq_tensor_fiber_plan(const hq_tensor* t, int mode, uint64_t* units, uint64_t* long_nnz, uint64_t* segments,
                         uint64_t* short_max);
/* sorted, merged entries (sparse_tensor.hpp:44-51): coords nnz*order, values nnz */
int hq_tensor_export(const hq_tensor* t, uint32_t* coords, double* values);
/* ModeBuckets (sparse_tensor.hpp:25-32): offsets dims[mode]+1, entries nnz */
int hq_tensor_buckets(const hq_tensor* t, int mode, uint64_t* offsets, uint64_t* entries);
/* norm_sq(const SparseTensor&) (sparse_tensor.hpp:69; sparse_tensor.cpp:91-95) */
int hq_tensor_norm_sq(const hq_tensor* t, double* out);

/* ------------------------------------------------------------------ .tns --
 * load_tns (sparse_tensor.hpp:76-79; sparse_tensor.cpp:136-215): the text parse
 * split over host threads with the reference's rules and errors (PARSE with
 * the line as payload, RANGE / VALUE with the line in the message).
 * override_order 0 = no dims override.  The parsed COO stays in the handle:
 * query its size, copy it out, or build the device tensor from it. */
typedef struct hq_tns hq_tns;
int hq_tns_parse(const char* text, uint64_t len, int override_order, const uint64_t* override_dims, hq_tns** out);
int hq_tns_parse_file(const char* path, int override_order, const uint64_t* override_dims, hq_tns** out);
int hq_tns_info(const hq_tns* p, int* order, uint64_t* dims, uint64_t* nnz);
int hq_tns_copy(const hq_tns* p, uint32_t* coords, double* values);
int hq_tns_tensor(const hq_tns* p, void* stream, hq_tensor** out);
int hq_tns_destroy(hq_tns* p);

/* --------------------------------------------------------------- kernels --
 * ttmc_core (kernels.hpp:46; kernels.cpp:40-84): core = X x {U^T}. */
int hq_ttmc_core(const hq_tensor* t, const double* const* factors, const uint64_t* ranks,
                 double* core_out);
/* ttmctc_elementwise (kernels.hpp:52-54) and ttmctc_matrix (kernels.hpp:59-60):
 * A = Y_(n) G_(n)^T.  `core` may be NULL (then it is computed from the factors,
 * kernels.cpp:92-101).  `variant` 0 = element-wise, 1 = matrix; both map to
 * the same device kernel (same linear map, results agree to 1e-11,
 * kernels_test.cpp:167-190). */
int hq_ttmctc(const hq_tensor* t, const double* const* factors, const uint64_t* ranks,
              int mode, const double* core, int variant, double* a_out);

/* ------------------------------------------------------------ dense core --
 * qr_orthonormal (dense_core.hpp:60; dense_core.cpp:127-198): orthonormal basis
 * of col(A) with R_kk >= 0.  CholeskyQR2 on the device; a device Householder
 * QR with the reference's seeded rank-deficiency fill when CholeskyQR2 would
 * lose accuracy.  SHAPE if rows < cols. */
int hq_qr_orthonormal(uint64_t rows, uint64_t cols, const double* a, double* q_out);
/* subspace_distance (manifold.hpp:34-36; manifold.cpp:55-60) */
int hq_subspace_distance(uint64_t rows, uint64_t cols, const double* u, const double* v,
                         double* out);
/* random_factors (solvers.hpp:72-73; solvers.cpp:182-195): seeded Gaussian
 * (bit-exact tucker::Rng stream, generated on the host), QR on the device. */
int hq_random_factors(int order, const uint64_t* dims, const uint64_t* ranks, uint64_t seed,
                      double* const* factors_out);

/* ---------------------------------------------------------------- solver --
 * SolverConfig (solvers.hpp:17-28).  init: 0 random (seeded), 1 HOSVD (not
 * supported on this engine: returns CAPACITY beyond the desk-scale cap and
 * SHAPE otherwise... see DESIGN.md), 2 caller-supplied factors. */
typedef struct hq_config {
    int order;
    uint64_t ranks[8];
    uint64_t max_sweeps;      /* default 100 */
    double tol_fit_change;    /* default 1e-12 */
    uint64_t seed;
    int init;                 /* 0 random, 1 HOSVD (desk-scale, capacity-capped), 2 = use init_factors */
    int kernel;               /* 0 element-wise, 1 matrix (same device path) */
    int trace_gradients;      /* per-update diagnostics (ModeUpdateRecord), on the device */
    double tol_grad;          /* gradient stop sqrt(sum grad) <= tol_grad f, implies tracing */
    uint64_t capacity_cap;    /* dense unfolding cap in entries (kernels.hpp:62), default 2^31 */
} hq_config;

void hq_config_default(hq_config* cfg);

/* IterationTrace (solvers.hpp:37-63), caller-allocated for max_sweeps sweeps.
 * With trace_gradients (or tol_grad > 0) the per-update ModeUpdateRecords
 * (solvers.hpp:40-49) are filled for update i = (sweep - 1) * order + mode:
 * f_before / f_after / elapsed_s [max_sweeps * order], sigma / lambda
 * [max_sweeps * order * sigma_stride] (first K_mode entries, descending). */
typedef struct hq_trace {
    double data_norm_sq;
    double initial_objective;
    uint64_t sweeps;           /* filled */
    double* objective;         /* [max_sweeps] */
    double* fit;               /* [max_sweeps] */
    double* drift;             /* [max_sweeps * order] */
    double* grad_norm_sq;      /* [max_sweeps * order] or NULL (zeros unless tracing) */
    double* elapsed_s;         /* [max_sweeps] or NULL: cumulative device time */
    double* upd_f_before;      /* or NULL */
    double* upd_f_after;       /* or NULL */
    double* upd_elapsed_s;     /* or NULL: device time between successive updates' diagnostics points */
    double* upd_sigma;         /* or NULL: singular values of A^(n) */
    double* upd_lambda;        /* or NULL: eigenvalues of G_(n) G_(n)^T */
    uint64_t sigma_stride;     /* caller: row stride of upd_sigma / upd_lambda (>= max rank) */
    uint64_t updates;          /* filled: number of update records (0 unless tracing) */
} hq_trace;

/* hoqri (solvers.hpp:80; solvers.cpp:50-178, 217-219): the whole solve on the
 * device.  factors_out: N host buffers; core_out: prod K doubles. */
int hq_hoqri(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors,
             double* const* factors_out, double* core_out, hq_trace* trace);

/* ------------------------------------------------------------- harness --
 * bench_kernel (harness.hpp:75-82; harness.cpp:350-381): `repetitions` TTMcTC
 * calls of `mode` on a fixed state, each timed on the device with CUDA events
 * (the G_(n)^T build and the fused pass, factors and core already resident);
 * seconds_out[repetitions]; transient_bytes[2] = the call's device scratch,
 * total and largest single buffer (the meter's counterpart, kernels.hpp:15-41). */
int hq_bench_ttmctc(const hq_tensor* t, const double* const* factors, const uint64_t* ranks, int mode,
                    uint64_t repetitions, double* seconds_out, uint64_t* transient_bytes);
/* gen_synthetic (harness.hpp:27-31; harness.cpp:62-98), bit-identical stream:
 * coords_out nnz * order, values_out nnz.  INFEASIBLE when nnz exceeds the
 * cells.  Host only (no device needed). */
int hq_gen_synthetic(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, uint32_t* coords_out,
                     double* values_out);

/* ---------------------------------------------------------- desk-scale --
 * The reference's dense paths, on the device (capacity-capped like the
 * reference: CAPACITY when rows > cap / cols):
 *  densify_unfold (kernels.hpp:70-71): X_(n) dense, out I_n x prod_{v!=n} I_v;
 *  ttmc_unfold_dense (kernels.hpp:66-67): Y_(n) dense, out I_n x prod_{v!=n} K_v;
 *  svd_leading (dense_core.hpp:64): leading k left singular vectors of a
 *    rows x cols host matrix (cuSOLVER eigen-solve of the smaller Gram side;
 *    equal to the reference's as a subspace, signs may differ);
 *  init_factors (solvers.hpp:69-70): random, HOSVD or error per cfg->init;
 *  hooi (solvers.hpp:82-83; solvers.cpp:93-178): same trace contract as hq_hoqri. */
int hq_densify_unfold(const hq_tensor* t, int mode, uint64_t capacity_cap, double* out);
int hq_ttmc_unfold_dense(const hq_tensor* t, const double* const* factors, const uint64_t* ranks, int mode,
                         uint64_t capacity_cap, double* out);
int hq_svd_leading(uint64_t rows, uint64_t cols, const double* y, uint64_t k, double* u_out);
/* jacobi_eig_sym (dense_core.hpp:85-90): eigenpairs of the symmetrised n x n
 * host matrix, values descending, eigenvector j in column j of the row-major
 * `vectors` (may be NULL); cuSOLVER syevd on the device, so vector signs may
 * differ from the reference's Jacobi rotations */
int hq_sym_eig(uint64_t n, const double* m, double* values_desc, double* vectors);
int hq_init_factors(const hq_tensor* t, const hq_config* cfg, double* const* factors_out);
int hq_hooi(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors,
            double* const* factors_out, double* core_out, hq_trace* trace);

/* fit_error (solvers.hpp:87; solvers.cpp:225-236) */
int hq_fit_error(double data_norm_sq, uint64_t core_size, const double* core, double* out);

/* ------------------------------------------------ device-resident solver --
 * The same solve, split so that a benchmark can keep every operand in HBM and
 * time sweeps and single kernels on its own stream. */
typedef struct hq_solver hq_solver;

int hq_solver_create(const hq_tensor* t, const hq_config* cfg,
                     const double* const* init_factors, void* stream, hq_solver** out);
int hq_solver_destroy(hq_solver* s);
/* runs `sweeps` sweeps asynchronously on the solver's stream (CUDA graph) */
int hq_solver_run(hq_solver* s, uint64_t sweeps);
/* waits, checks the device status word, and reports a DEGENERATE error */
int hq_solver_sync(hq_solver* s);
/* launches only the fused sparse mode pass (TTMcTC + Gram + core projection)
 * for `mode` on the solver's stream: the dominant kernel, for timing */
int hq_solver_launch_mode_pass(hq_solver* s, int mode);
/* launches only the TTMcTC kernel for `mode` (A written to device scratch) */
int hq_solver_launch_ttmctc(hq_solver* s, int mode);
/* device status word after a sync (out: 8 slots): out[0] sweeps completed,
 * out[1] mode updates that took the Householder fallback, out[2] abort code
 * (0 running, 1 degenerate, 2 stopped, 3 multi-GPU fallback pending), out[3]
 * degenerate mode, out[4] mode updates that ran shifted CholeskyQR3, out[5]
 * multi-GPU updates finished by the host-driven Householder continuation,
 * out[6] 1 when the multi-GPU apply stores U_new straight into the other
 * ranks' replicas over peer memory (fused apply + all-gather), out[7] 0 */
int hq_solver_status(hq_solver* s, int64_t* out);
/* number of device kernels one sweep launches */
int hq_solver_launches_per_sweep(const hq_solver* s, uint64_t* out);
int hq_solver_download(hq_solver* s, double* const* factors_out, double* core_out, hq_trace* trace);
/* algorithmic work of one mode pass: flops and bytes (DESIGN.md roofline) */
int hq_solver_mode_pass_work(const hq_solver* s, int mode, double* flops, double* bytes);
int hq_solver_ttmctc_work(const hq_solver* s, int mode, double* flops, double* bytes);

/* ------------------------------------------------------------- multi-GPU --
 * One process per GPU.  Every rank builds the same tensor;
 * for each mode the unfolding's rows are split into contiguous whole-row
 * ranges of ~nnz/P nonzeros (the row partition of SPEC.md:247), each rank
 * runs the pass on its rows, K x K / K x L partials are all-reduced and new
 * factor rows broadcast from their owners (NCCL, captured in the sweep
 * graph).  The reference has no multi-GPU path; this is the north_star's. */
typedef struct hq_comm hq_comm;

/* NCCL unique id (128 bytes) — call on one rank, share with the others */
int hq_nccl_unique_id(uint8_t* id_out);
/* communicator on the current CUDA device; world 1 needs no NCCL */
int hq_comm_create(int world, int rank, const uint8_t* id, hq_comm** out);
int hq_comm_destroy(hq_comm* c);
/* the host transport: ranks on one node (any GPUs, or one shared GPU) exchange
 * through the POSIX shared-memory segment `name` ("/..." , created by the first
 * rank to attach); `capacity` = the largest collective in doubles (max I_n K_n).
 * Collectives are D2H copy -> host combine in rank order -> H2D copy on the
 * solver's stream; no kernel waits on another rank. */
int hq_comm_create_host(int world, int rank, const char* name, uint64_t capacity, hq_comm** out);
/* row-partitioned storage: keep only this rank's rows of every mode stream (the
 * solver's partition); the tensor is then usable only with a
 * distributed solver on the same communicator layout */
int hq_tensor_shard(hq_tensor* t, const hq_comm* comm);
/* host planner: rank r owns rows [bounds[r], bounds[r+1]) given a mode's
 * bucket offsets (length rows + 1); bounds has world + 1 slots */
int hq_partition_rows(const uint64_t* offsets, uint64_t rows, int world, uint64_t* bounds);
/* hq_solver_create on a communicator: the device-resident solve, distributed */
int hq_solver_create_dist(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors, void* stream,
                          const hq_comm* comm, hq_solver** out);

#ifdef __cplusplus
}
#endif

#endif /* HOQRI_B200_H */
