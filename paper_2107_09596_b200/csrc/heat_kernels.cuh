// heat_kernels.cuh -- host/device interface of the Heat1D Phi kernels.
//
// Phi for problems::Heat1D (reference heat1d.cpp:47-100) is a backward-Euler
// step: S sub-steps of a constant-coefficient tridiagonal solve
// (I + sub_dt L) x = rhs, optionally preceded by the manufactured forcing
// x += theta(t) * sin(pi x).  The reference runs the Thomas recurrences
// serially per vector; here one CTA owns one state vector (one time point)
// in registers, in a blocked arrangement (thread t holds elements
// [t*L, t*L+L)).  See heat_phi5.cu for the algorithm.
#pragma once

#include <cuda.h>
#include <cstdint>
#include <vector>

namespace atm {

constexpr int kMaxThreads = 512;
constexpr int kMaxWarps = kMaxThreads / 32;
constexpr int kMaxL = 32;
constexpr int kMaxCluster = 16;  // CTAs per cluster row (heat1d n <= 16 x 4096; past 8: non-portable clusters)
constexpr int kScanPerThread = 18;  // Mf[5], Pf_ex, Mb[5], Pb_ex, SB, q0, cfw, cbw, pad, cbwr

// Device view of one level's Phi coefficients.
//
// The tridiagonal matrix T = tridiag(a, b, a) (a = -r, b = 1 + 2r) equals
// the constant-coefficient LU product M = L_c U_c built from the fixed point
// (c*, d*) of the Thomas recurrence everywhere except entry (0,0):
//     T = M + delta e0 e0^T,  delta = a c*.
// Phi is therefore computed as x = M^{-1} b - s w with w = M^{-1} e0,
// s = sigma x0, x0 = (M^{-1} b)_0, sigma = delta / (1 + delta w0)
// (Sherman-Morrison: g . b = (M^{-1} b)_0 for g = M^{-T} e0).  On every
// thread's chunk w lies in span{q, p_b} -- the two vectors the blocked solve
// already combines -- so the correction only shifts the chunk's two carry
// coefficients by (-s) * (cfw, cbw).  w decays geometrically from index 0:
// only the first `ncw` warps apply it.
struct HeatCoefDev {
    const double* scan;    // [nt][16] per-thread scan multipliers + (cfw, cbw)
    const double* wf;      // [kMaxWarps][kMaxWarps] cross-warp carry weights (forward)
    const double* wb;      // [kMaxWarps][kMaxWarps] (backward)
    const double* wk;      // [kMaxWarps][kMaxWarps] forward-into-backward coupling weights
    const double* powc;    // [3][kMaxL] q, p_b of interior threads; q of the padded last thread
                           // (sb_m > 0: the two q rows hold one table per sub-block)
    const double* theta;   // [np*S] forcing amplitude per (index, substep) or null
    const double* prof;    // [nt*L] forcing profile sin(pi x_i) or null
    double beta_c, gamma_c, cneg_c;  // fixed-point factors: 1/d*, r/d*, -c*
    double sigma;          // Sherman-Morrison scale
    int ncw;               // warps [0, ncw) carry the left correction vector
    // sub-block local passes (plain heat rows with L = 16): every chunk runs as
    // L / sb_m independent chains of sb_m elements; sb_af = gamma^sb_m and
    // sb_ab = (-c)^sb_m carry between the sub-blocks (heat_phi5.cu, tri_solve_sb)
    int sb_m;
    double sb_af, sb_ab;
    // the interior sub-block's q and p_b, read as constant-bank operands (no
    // shared-memory table reads in the fix-up); the thread holding element
    // n-1 folds its shorter sub-blocks into its c_b (powc row 2: kappa_b)
    double sb_q[8], sb_pb[8];
    int ncw_r0;            // cyclic: warps [ncw_r0, nw) carry the right one
    // cyclic (periodic) matrices: Woodbury capacitance S (2x2) and the
    // x_{n-1} pick-up of thread tl (element pl-1)
    int cyclic, tl, pl;
    double S[4], ql, pbl;
    const double* xw;      // [4][kMaxWarps] x0 / xn weights of the warp totals
    // Allen-Cahn Newton (prob == 1): F(u) = u - dt (c D2 u + u - u^3) - u_prev
    int prob;              // 0 heat, 1 Allen-Cahn
    int newton_max;
    double ac_dt, ac_c, ac_shift, newton_tol, ac_umax2, inner_eta;
    int* fail;             // set to 1 when Newton hits newton_max
    int n, pitch, nt, L;
    int substeps;
    // rows split over a cluster of `cl` CTAs (n > 5376): CTA q of the cluster
    // holds elements [4096 q, 4096 q + 4096) of every row (nt = 128, L = 32);
    // the tables above are per block, concatenated ([cl][...]); blk: per-block
    // ncw, ncw_r0, tl, pl, ql, pbl (8 doubles each); cS: the 2cl x 2cl
    // Woodbury matrix coupling the blocks (heat_phi5.cu, cluster rows)
    int cl;
    const double* blk;
    const double* cS;
};

// Host-side construction of a level's coefficients (heat1d.cpp:24-45).
struct HeatLevelHost {
    std::vector<double> scan, wf, wb, wk, powc, xw;
    // cyclic: first / last entries of wl = M^{-1} e_0 and wr = M^{-1} e_{n-1}
    long double w0 = 0, wn = 0, wr0 = 0, wrn = 0;
    // cluster rows: per-block scalars and the coupling matrix (HeatCoefDev)
    std::vector<double> blk, cS;
    double r = 0, beta_c = 0, gamma_c = 0, cneg_c = 0, sigma = 0;
    double S[4] = {0, 0, 0, 0}, ql = 0, pbl = 0;
    int sb_m = 0;
    double sb_af = 0, sb_ab = 0, sb_q[8] = {0}, sb_pb[8] = {0};
    int cyclic = 0, ncw_r0 = 0, tl = 0, pl = 0;
    double fit_err = 0;  // max |w - (cfw q + cbw p_b)| / max |w| over the correction chunks
    int ncw = 0, n = 0, pitch = 0, nt = 0, L = 0, substeps = 1;
};
// r = sub_dt/h^2 (a = -r, diagonal 1 + 2r + shift); cyclic: periodic corners
HeatLevelHost heat_level_host(int n, int pitch, int L, double r, double shift, int substeps,
                              bool cyclic);
// rows of n > 5376 split over cl CTAs of 4096 elements (L = 32, 128 threads
// each): per-block tables concatenated, and the block coupling
HeatLevelHost heat_cluster_host(int n, int cl, double r, int substeps);

// Job kinds of the sweep kernel (one job per C-point index J of a level).
enum SweepKind { SW_F = 0, SW_FCF = 1, SW_CRELAX = 2, SW_RESID = 3 };
// TAIL_BOTH: the residual row is stored (next cycle's restriction input)
// and its square sum written (this cycle's stopping norm)
enum TailKind { TAIL_NONE = 0, TAIL_STORE = 1, TAIL_SQ = 2, TAIL_BOTH = 3 };
enum StoreKind { STORE_NONE = 0, STORE_ALL = 1, STORE_CF = 2 };
__host__ __device__ inline bool store_row(int mode, int i, int m) {
    return mode == STORE_ALL || (mode == STORE_CF && (i % m == 0 || (i + 1) % m == 0));
}

struct SweepArgs {
    HeatCoefDev co;
    int kind;          // SweepKind
    int m, np;         // level CF split (m = 1 => every point is a job)
    int j0, j1;        // job range [j0, j1)
    int u_base;        // global index of row 0 of the u array
    int g_base;        // global index of row 0 of the g array
    int add_g;         // u_i = Phi(u_{i-1}) + g_i with g stored per point
    int forced;        // Phi includes forcing (folded manufactured)
    int store;         // STORE_ALL, or STORE_CF: only C rows and the last F row of
                       // each interval (the rest are rewritten by the cycle's
                       // correction F-sweep before anything reads them)
    int tail;          // TailKind: residual at the next C-point
    int out_base;      // global (coarse) index of row 0 of the tail target
    double* sq;        // squares (TAIL_SQ) at (tail point - sq_base) / sq_div
    int sq_base;
    int sq_div;        // 1: per-point array; m: per-C-point array (stopping norm)
    int n_out;         // output staging buffers (1 or 2)
    int u_div;         // > 1: the u array holds only the C points (row = (i - u_base) / u_div)
    int st_hint;       // L2 policy of the per-warp row stores: 0 default, 1 evict_first, 2 evict_last
};

enum WindowKind { WK_LINEAR = 0, WK_FAS = 1, WK_FORWARD = 2, WK_APPLY = 3, WK_FAS_RHS = 4 };

struct WindowArgs {
    HeatCoefDev co;
    int kind;
    int k;             // window distance
    int pre_lo, pre_e0, pre_e1;  // prefix job (chain from pre_lo) emitting [pre_e0, pre_e1]; pre_e1 < pre_e0 => none
    int p0, p1;        // individual windows p in [p0, p1]
    int x1_base, x2_base, x3_base, out_base;
    int out_stride;    // emit row for p: out index p*out_stride (linear: fine m)
    int forced;        // Phi includes forcing theta*prof
    int seed_zero;     // WK_APPLY: seed is the zero vector (forcing computation)
    int idx0;          // WK_APPLY: step index offset (job p applies Phi_{idx0+p})
    int seed_off;      // WK_APPLY: seed row is p + seed_off
    int two_s;         // WK_LINEAR: double-buffered fine C rows (long prefix chain)
};

// Launchers (stream-ordered).  Return cudaError_t as int.
int launch_heat_sweep(const SweepArgs& args, const CUtensorMap& tm_u, const CUtensorMap& tm_g,
                      const CUtensorMap& tm_out, const CUtensorMap& tm_uw,
                      const CUtensorMap& tm_outw, int grid, cudaStream_t s);
int launch_heat_window(const WindowArgs& args, const CUtensorMap& tm_x1, const CUtensorMap& tm_x2,
                       const CUtensorMap& tm_x3, const CUtensorMap& tm_out, int grid,
                       cudaStream_t s);
size_t heat_sweep_smem(const SweepArgs& a);
size_t heat_window_smem(const WindowArgs& a);
// max resident CTAs per SM for the kernel that would serve these args
int heat_sweep_occupancy(const SweepArgs& a);
int heat_window_occupancy(const WindowArgs& a);

}  // namespace atm
