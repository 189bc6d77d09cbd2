// hq_long.cuh — arguments of the DMMA long-row kernels (hq_long.cu).
#pragma once

#include "hq_plan.cuh"

namespace hq {

struct LongArgs {
    uint64_t rbase, rows;            // processed row range of the mode (multi-GPU share)
    const int64_t* rowptr;
    const double* val;
    const uint32_t* i0;              // other-mode index streams (ascending v != n)
    const uint32_t* i1;
    const uint32_t* i2;              // order 4 only
    const double* u0;                // matching factors
    const double* u1;
    const double* u2;
    const double* un;                // U_n (kCore)
    const double* gt;                // G_(n)^T, L x K_n (kTTMcTC)
    const uint32_t* long_ids;
    const int64_t* long_segptr;
    const int64_t* seg_begin;
    const uint32_t* seg_row;
    uint64_t nlong, nseg;
    double* ypart;                   // [nseg][L]
    double* A;
    double* mpart;
    double* wpart;
    double* maxpart;
    int kind;
    int slot0;
    const DevStatus* st;
    int run_if;
    int l1_0, l1_1, l1_2;            // L1-allocating gathers for hot (skewed) factors (ModeLayout::hot)
};

bool long_fast_supported(const ModeShape& sh);
// segment kernel grid: min(segments, SMs x resident CTAs); fix-up grid given
void launch_long_fast(const LongArgs& a, const ModeShape& sh, int fix_grid, cudaStream_t s);

}  // namespace hq
