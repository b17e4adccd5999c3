// common_kernels.cuh -- elementwise / reduction kernels shared by every Phi
// family, and the scalar (n = 1) Phi backend (Dahlquist, scalar fixture).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace atm {

// Scalar Phi: v = mult * u (+ ff[index] when folded on level 0):
// dahlquist.hpp:25-30 (mult includes sub-steps, :36-42) and the
// tests/support.hpp:35-41 fixture.
struct ScalarCoefDev {
    double mult;
    const double* ff;   // folded fine forcing on level 0, or null
};

struct ScalarSweepArgs {
    ScalarCoefDev co;
    int kind, m, np, j0, j1;
    double* u; int u_base;
    const double* g; int g_base; int add_g;
    int store, tail;
    double* out; int out_base;
    double* sq; int sq_base; int sq_div;  // squares at (tail point - sq_base) / sq_div
    int u_div;  // > 1: C-point-only u array
};

struct ScalarWindowArgs {
    ScalarCoefDev co;
    int kind, k;
    int pre_lo, pre_e0, pre_e1, p0, p1;
    const double* x1; int x1_base;
    const double* x2; int x2_base;
    const double* x3; int x3_base;
    double* out; int out_base; int out_stride;
    int seed_zero, idx0, seed_off;
};

int launch_scalar_sweep(const ScalarSweepArgs& a, cudaStream_t s);
int launch_scalar_window(const ScalarWindowArgs& a, cudaStream_t s);

// u[row i][q] = random_state(seed + i, n)[q] for i in [i0, i1) (i >= 1),
// bitwise equal to state_vector.hpp:108-118.
int launch_fill_random(double* u, int base, int pitch, int n, int i0, int i1, uint64_t seed,
                       cudaStream_t s, int step = 1);
// rows [i0,i1) := v (n values, device)
int launch_fill_rows(double* u, int base, int pitch, int n, int i0, int i1, const double* v,
                     cudaStream_t s);
// r = g - u elementwise for one row; optional square sum into sq[0]
int launch_row_diff(double* r, const double* g, const double* u, int n, double* sq,
                    cudaStream_t s);
// FAS correction u[c_j] += cu[j] - cv[j] for j in [j0, j1) (solver.cpp:285-289)
int launch_c_correct(double* u, int u_base, int m, const double* cu, const double* cv,
                     int c_base, int pitch, int n, int j0, int j1, cudaStream_t s);
// g_0 = v_0 + r_0 (solver.cpp:209-211)
int launch_row_sum(double* g, const double* v, const double* r, int n, cudaStream_t s);
// out[0] = sqrt(sum_i sq[i]) with a fixed association (shard-count independent)
int launch_norm_from_squares(const double* sq, int count, double* out, cudaStream_t s);
// FunctionalChange norm (solver.cpp:380-396), one warp per level-0 C point j in
// [j0, j1): f_j = w.u (w != NULL) or u.norm2() (w == NULL, the reference CLI's
// functional, run_config.cpp:241-243); unless init, rel_j = |f_j - prev_j| /
// max(|prev_j|, 1e-300) and *out_max = max_j rel_j (zeroed first; a NaN ratio
// never raises it, as with std::max); then prev_j := f_j (prev indexed by j).
int launch_functional(const double* u, int u_base, int m, int pitch, int n, const double* w,
                      double* prev, int j0, int j1, double* out_max, int init, cudaStream_t s);

}  // namespace atm
