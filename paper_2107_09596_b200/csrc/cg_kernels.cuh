// cg_kernels.cuh -- 2D heat Phi (BASELINE configs 2 and 4): backward Euler
// with the 5-point Laplacian (zero Dirichlet), each sub-step solved by
// matrix-free CG to |r| <= rtol |b| from x0 = u_prev.  No reference Phi
// exists; the restatement is oracle/atm_oracle.c h2_solve.
//
// One system is owned by a thread-block cluster of `cs` CTAs; CTA q holds
// rows [q R, q R + R) of the nx x nx grid.  The search direction p lives in
// shared memory with one halo row above and below (read from the
// neighbouring CTAs through DSMEM); x and r live in shared memory when they
// fit (clusters of up to 4 CTAs), else in two global scratch rows per
// cluster (L2-resident).  Dot products are fixed-order CTA sums followed by a
// rank-ordered cluster sum, so every CTA holds bitwise the same alpha/beta.
#pragma once

#include <cuda_runtime.h>

namespace atm {

struct CgCoefDev {
    int nx, n, pitch;
    int cs, R;            // CTAs per system (cluster size), grid rows per CTA
    double c, diag;       // c = sub_dt / h^2, diag = 1 + 4c
    double sdt;           // sub-step
    const double* src;    // source f (n values) or null
    int substeps;
    double rtol;
    int cg_max;
    int* fail;            // set to 1 when CG hits cg_max
    unsigned long long* iters;  // running count of inner (CG / BiCGSTAB) iterations, or null
    int x_smem;           // x and r in shared memory (else xg)
    double* xg;           // global scratch: x, r rows per cluster slot
    int E;                // 0: generic kernel; > 0: register variant, E elements per thread;
                          // 1000 + e: strip kernel, e grid rows per thread (see heat2d_cg.cu)
    int nt;               // threads per CTA
    int strip;            // 1: strip kernel (one-barrier Chronopoulos-Gear CG, vectors in registers)
    int sWX, sWY;         // strip kernel: warps across a row (32 columns each), warp-rows per CTA
    // strip kernel, group mode (systems too large for one 16-CTA cluster):
    // cs CTAs of a cooperative grid per system, exchanging through global
    // memory (gex: per group rows + partials, gflag: per CTA sequence flags);
    // p and s in shared memory
    int glob;
    double* gex;
    unsigned long long* gflag;
    // Gray-Scott (prob == 1): periodic nx x nx cells, state [u; v]; one CTA
    // per system, every work vector in shared memory
    int prob;
    double gs_h2inv, gs_du, gs_dv, gs_feed, gs_kill, gs_linear_tol;
    int gs_reaction, gs_bounds_check;
    double gs_bound_lo, gs_bound_hi, newton_tol;
    int newton_max;
};

// same job semantics as ScalarSweepArgs / the heat sweep kernel
struct CgSweepArgs {
    CgCoefDev co;
    int kind, m, np, j0, j1;
    double* u; int u_base;
    const double* g; int g_base; int add_g;
    int forced, store, tail;
    double* out; int out_base;
    double* sq; int sq_base; int sq_div;  // squares at (tail point - sq_base) / sq_div
    int u_div;  // > 1: C-point-only u array
};

struct CgWindowArgs {
    CgCoefDev co;
    int kind, k;
    int pre_lo, pre_e0, pre_e1, p0, p1;
    const double* x1; int x1_base;
    const double* x2; int x2_base;
    const double* x3; int x3_base;
    double* out; int out_base; int out_stride;
    int forced, seed_zero, idx0, seed_off;
};

// host: cluster geometry for an nx x nx system (cs, R, E, nt, x placement)
void cg_geometry(int nx, CgCoefDev& co);
// host: Gray-Scott geometry (one CTA, 10 state-size vectors in smem); false
// when 2 nx^2 does not fit
// Gray-Scott; cs: CTAs per system when the work vectors live in global
// scratch (few concurrent systems: more SMs per Phi)
bool gs_geometry(int nx, CgCoefDev& co, int cs = 1);
size_t cg_smem_bytes(const CgCoefDev& co);
// group mode: doubles of exchange area per group (gex), flags per group = cs
size_t cg_glob_doubles_per_group(const CgCoefDev& co);
// clusters that can be resident at once (the number of x scratch rows needed)
int cg_max_clusters(const CgCoefDev& co);
int launch_cg_sweep(const CgSweepArgs& a, cudaStream_t s);
int launch_cg_window(const CgWindowArgs& a, cudaStream_t s);

}  // namespace atm
