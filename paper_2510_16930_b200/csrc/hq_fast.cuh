// hq_fast.cuh — arguments of the specialised order-3 pass (hq_pass_fast.cu).
#pragma once

#include "hq_plan.cuh"

namespace hq {

struct FastArgs {
    uint64_t rbase;  // first row of the processed range
    uint64_t rows;   // rows in the range
    const int64_t* rowptr;
    const double* val;
    const uint32_t* ia;   // first other mode's index
    const uint32_t* ib;   // second other mode's index
    const double* ua;     // factor of the first other mode  (I_a x K_a)
    const double* ub;     // factor of the second other mode (I_b x K_b)
    const double* un;     // U_n (kCore)
    const double* gt;     // G_(n)^T, L x K_n (kTTMcTC)
    double* A;
    double* mpart;
    double* wpart;
    double* maxpart;
    int kind;
    int slot0;
    const DevStatus* st;
    int run_if;
    int a_only;           // standalone TTMcTC (kTTMcTCOnly): A only, no M / W partials
    int l1_a, l1_b;       // L1-allocating gathers for a hot (skewed) factor (ModeLayout::hot)
    int short_max;        // rows with more nonzeros are long rows (ModeLayout::short_max <= kShortMax)
};

void debug_phase_cycles(unsigned long long* out, int reset);

bool fast_supported(const ModeShape& sh);
int fast_grid(int ka, int kb, int kn);
void launch_fast(const FastArgs& a, const ModeShape& sh, int grid, cudaStream_t s);

}  // namespace hq
