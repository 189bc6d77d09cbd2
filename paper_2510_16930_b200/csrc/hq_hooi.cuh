// hq_hooi.cuh — desk-scale dense paths (hq_hooi.cu): HOSVD init and HOOI.
#pragma once

#include "hq_plan.cuh"
#include "hoqri_b200.h"

namespace hq {

double max_abs_dev(const double* v, uint64_t n, cudaStream_t s);
uint64_t densify_cols(const DeviceTensor& T, int mode);
void densify_unfold_dev(const DeviceTensor& T, int mode, uint64_t cap, DBuf<double>& out, cudaStream_t s);
void ttmc_unfold_dense_dev(const DeviceTensor& T, int mode, const FactorPtrs& f, const int* ranks, uint64_t cap,
                           DBuf<double>& y, cudaStream_t s);
// u_out: m x k device, y: m x p device
void svd_leading_dev(const double* y, uint64_t m, uint64_t p, int k, double* u_out, cudaStream_t s);
// symmetric eigenpairs of a host n x n matrix (descending; vectors row-major, may be null)
void sym_eig_host(uint64_t n, const double* m, double* values_desc, double* vectors, cudaStream_t s);
// HOSVD (solvers.cpp:202-215) into device factor buffers U[v] (I_v x K_v)
void hosvd_init_dev(const DeviceTensor& T, const int* ranks, uint64_t cap, double* const* U, cudaStream_t s);
// the HOOI solve (solvers.cpp:50-178 with Algorithm::kHooi)
void hooi_solve(const DeviceTensor& T, const hq_config& cfg, const double* const* init_host,
                double* const* factors_out, double* core_out, hq_trace* tr, cudaStream_t s);

// provided by hq_solver.cu
void ttmc_core_dev(const DeviceTensor& T, const FactorPtrs& f, const int* ranks, double* core, cudaStream_t s);
double subspace_distance_dev(const double* u, const double* v, uint64_t rows, int k, cudaStream_t s);
double orthonormality_defect_dev(const double* u, uint64_t rows, int k, cudaStream_t s);
void init_factors_dev(const DeviceTensor& T, const hq_config& cfg, const double* const* init_host, double* const* U,
                      cudaStream_t s);

}  // namespace hq
