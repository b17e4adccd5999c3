/*
 * atm_oracle.h -- CPU restatement of the AT-MGRIT reference path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2107_09596_b200/) links, loads or calls this code.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
 * it, and only as the checker.
 *
 * Every function restates the algorithm of the reference `tempo` library
 * (/root/reference/proj) in plain C over flat point-major arrays; the
 * comment above each definition in atm_oracle.c cites the reference
 * file:line it follows.  The restatement is pinned against (a) the
 * reference's own known-answer tests, restated in tests/test_oracle_*.py,
 * and (b) fixtures produced by the compiled reference itself
 * (oracle/_ref/tempo_ref, built by oracle/Makefile from the reference
 * sources in place), committed under tests/golden/.
 */
#ifndef ATM_ORACLE_H
#define ATM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAXL 8

enum { ORC_OK = 0, ORC_NOT_CONVERGED = 1, ORC_CONFIG = 2, ORC_FAULT = 3,
       ORC_DIVERGED = 4, ORC_NONLINEAR = 5 };

enum { ORC_HEAT1D = 1, ORC_DAHLQUIST = 2, ORC_SCALAR = 3, ORC_ALLEN_CAHN = 4,
       ORC_HEAT2D = 5, ORC_GRAY_SCOTT = 6 };

enum { ORC_TWO_LEVEL = 0, ORC_VCYCLE = 1, ORC_NESTED_V = 2 };
enum { ORC_RELAX_F = 0, ORC_RELAX_FCF = 1 };
enum { ORC_NORM_L2 = 0, ORC_NORM_FUNCTIONAL = 1 };
enum { ORC_GUESS_CONSTANT = 0, ORC_GUESS_RANDOM = 1, ORC_GUESS_PROVIDED = 2 };

typedef struct orc_problem {
    int kind;
    int n;                 /* state size (ignored for scalar kinds: 1)       */
    int folded;            /* forcing convention (application.hpp:23-29)     */
    /* heat1d */
    double x0, x1;
    int manufactured;      /* heat1d.hpp:27                                  */
    /* dahlquist */
    double lambda, u0;
    /* scalar linear test fixture (tests/support.hpp:19-60) */
    int n_mult;
    double mult[ORC_MAXL];
    const double* fine_forcing;
    int n_ff;
    /* allen-cahn: u_t = eps^2 u_xx + u - u^3, periodic on [0, length) */
    double eps, length;
    double newton_tol;
    int newton_max;
    /* heat2d: u_t = lap(u) + f on the unit square, nx*nx interior */
    int nx;
    double cg_rtol;
    int cg_max;
    const double* source;  /* f on the interior grid, nx*nx (may be NULL)   */
    /* optional initial-condition override (n values)                       */
    const double* ic;
    /* gray-scott (gray_scott.hpp:24-38): n = nx cells per side, state [u; v]  */
    double gs_domain, gs_feed, gs_kill, gs_du, gs_dv, gs_linear_tol;
    int gs_reaction, gs_bounds_check;
    double gs_bound_lo, gs_bound_hi;
} orc_problem;

typedef struct orc_grid {
    double t0, tf;
    int n_points;
    int n_m;               /* number of coarsening factors (levels - 1)      */
    int m[ORC_MAXL];
    int k;
} orc_grid;

typedef struct orc_solver {
    int mode, relaxation, nu, max_iters;
    double tol;
    int norm;
    const double* functional_w;   /* linear functional w.u (n values)      */
    int initial_guess;
    uint64_t seed;
    const double* constant_value; /* n values or NULL (=> IC)               */
    const double* provided;       /* n_points*n values                      */
    int coarse_substeps;
} orc_solver;

typedef struct orc_driver orc_driver;

/* splitmix64 fill, state_vector.hpp:92-118 */
void orc_random_state(uint64_t seed, int n, double* out);

/* hierarchy, hierarchy.cpp:24-50 */
int orc_level_points(const orc_grid* g, int level);
double orc_level_dt(const orc_grid* g, int level);

orc_driver* orc_create(const orc_problem* p, const orc_grid* g, const orc_solver* s,
                       int* status);
const char* orc_error(const orc_driver* d);
const char* orc_create_error(void);
void orc_destroy(orc_driver* d);

int orc_setup(orc_driver* d);
int orc_cycle(orc_driver* d);
int orc_nested_init(orc_driver* d);
int orc_residual_norm(orc_driver* d, double* out);
/* drive(): history[] receives one norm per iteration (capacity max_iters) */
int orc_drive(orc_driver* d, double* history, int* iterations, int* converged);

int orc_n_levels(const orc_driver* d);
int orc_vector_size(const orc_driver* d);
/* which: 0=u 1=g 2=v 3=r; returns a pointer to [n_points_level * n] */
double* orc_array(orc_driver* d, int level, int which);

/* Application-level primitives (for kernel-level parity tests) */
int orc_step(orc_driver* d, int level, int index, const double* in, double* out);
int orc_forcing(orc_driver* d, int level, int index, double* out);
void orc_initial_condition(orc_driver* d, double* out);

/* kernels.cpp restatements over the driver's own arrays of `level` */
int orc_k_f_relax(orc_driver* d, int level, int first_interval, int count);
int orc_k_c_relax(orc_driver* d, int level, int first_c, int count);
int orc_k_residual(orc_driver* d, int level, int first, int count, double* r_out);
int orc_k_window_linear(orc_driver* d, int level, int lo, int size, const double* r_win,
                        double* out);
int orc_k_window_fas(orc_driver* d, int level, int lo, int size, const double* v_win,
                     const double* r_win, double* out);

#ifdef __cplusplus
}
#endif
#endif
