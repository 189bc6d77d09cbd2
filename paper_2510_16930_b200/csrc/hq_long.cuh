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
    // fiber units (order 3, FiberLayout): when ustart is set the segment kernel is k_fibseg -- rowptr, i0 and the
    // segment plan describe the unit stream, val / i1 stay the mode's nonzero streams, u1 the last factor
    const int64_t* ustart = nullptr; // units: first nonzero
    const uint8_t* ulen = nullptr;   // units: nonzeros (<= kFiberCap)
    const int64_t* rowptr_nz = nullptr;  // the mode's nonzero rowptr (rowptr is the unit rowptr)
    const int64_t* seg_cost = nullptr;  // nseg + 1 prefix costs: CTAs take segment ranges of equal cost
};

bool long_fast_supported(const ModeShape& sh);
void debug_fib_phase_cycles(unsigned long long* out, int reset);  // zeros unless built with -DHQ_PHASE_TIMING
// segment kernel grid: min(segments, SMs x resident CTAs); fix-up grid given
void launch_long_fast(const LongArgs& a, const ModeShape& sh, int fix_grid, cudaStream_t s);

}  // namespace hq
