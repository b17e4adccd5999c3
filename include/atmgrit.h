/*
 * atmgrit.h -- C ABI of the B200-native AT-MGRIT hot path.
 *
 * This is the drop-in boundary for the reference solver `tempo`
 * (/root/reference/proj).  Each entry point names the reference interface it
 * replaces (file:line relative to /root/reference/proj).  Plain C types only:
 * caller-owned host buffers in, library-owned device memory inside.  A
 * context is not thread-safe: one host thread drives one context.
 *
 * Status codes mirror the reference's error taxonomy
 * (include/tempo/errors.hpp:9-42) and CLI exit codes
 * (include/tempo/cli.hpp:12-17).
 */
#ifndef ATMGRIT_H
#define ATMGRIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATM_ABI_VERSION 6
#define ATM_MAX_LEVELS 8

typedef enum {
    ATM_OK = 0,
    ATM_NOT_CONVERGED = 1,  /* StopReason::MaxIterations (solver_config.hpp:31)      */
    ATM_CONFIG_ERROR = 2,   /* ConfigError (errors.hpp:9-13)                          */
    ATM_RUNTIME_FAULT = 3,  /* RuntimeFault (errors.hpp:27-35); CUDA/NCCL failures     */
    ATM_DIVERGED = 4,       /* DivergenceError (errors.hpp:15-25)                      */
    ATM_NONLINEAR_FAIL = 5  /* NonlinearSolveError (errors.hpp:37-41)                  */
} atm_status;

/* Phi families (the device-side descriptor that replaces the virtual
 * Application::step, application.hpp:33-76). */
typedef enum {
    ATM_PHI_HEAT1D = 1,     /* problems::Heat1D, heat1d.hpp:20-76                      */
    ATM_PHI_DAHLQUIST = 2,  /* problems::Dahlquist, dahlquist.hpp:12-50                */
    ATM_PHI_SCALAR = 3,     /* tests/support.hpp:19-60 ScalarLinear fixture           */
    ATM_PHI_ALLEN_CAHN = 4, /* new: BASELINE config 3 (no reference counterpart)       */
    ATM_PHI_HEAT2D = 5,     /* new: BASELINE configs 2, 4 (no reference counterpart)   */
    ATM_PHI_GRAY_SCOTT = 6  /* problems::GrayScott, gray_scott.hpp:12-68 (Newton +
                               Jacobi-preconditioned BiCGSTAB; nx = cells per side) */
} atm_phi_kind;

typedef enum { ATM_TWO_LEVEL = 0, ATM_VCYCLE = 1, ATM_NESTED_V = 2 } atm_mode;   /* CycleMode   */
typedef enum { ATM_RELAX_F = 0, ATM_RELAX_FCF = 1 } atm_relaxation;              /* Relaxation  */
typedef enum { ATM_NORM_L2 = 0, ATM_NORM_FUNCTIONAL = 1 } atm_norm;              /* NormKind    */
typedef enum { ATM_GUESS_CONSTANT = 0, ATM_GUESS_RANDOM = 1, ATM_GUESS_PROVIDED = 2 } atm_guess;
typedef enum { ATM_STORE_FULL = 0, ATM_STORE_CPOINTS = 1 } atm_storage;
/* FunctionalChange functional f(u) (SolverConfig::functional, solver_config.hpp:43):
 * LINEAR = w.u with functional_w; NORM2 = u.norm2() (state_vector.hpp:61-67),
 * the reference CLI's functional (run_config.cpp:241-243). */
typedef enum { ATM_FUNCTIONAL_LINEAR = 0, ATM_FUNCTIONAL_NORM2 = 1 } atm_functional;

/* Problem descriptor: replaces the Application subclass (application.hpp:33). */
typedef struct atm_problem {
    int kind;              /* atm_phi_kind                                          */
    int n;                 /* vector_size() (heat1d n_dof, allen-cahn nx)            */
    int folded;            /* forcing_folded() (application.hpp:23-29)               */
    double x0, x1;         /* heat1d interval (heat1d.hpp:25-26)                     */
    int manufactured;      /* heat1d manufactured_forcing (heat1d.hpp:27)            */
    double lambda, u0;     /* dahlquist (dahlquist.hpp:17)                           */
    int n_mult;            /* scalar fixture: multiplier per level                   */
    double mult[ATM_MAX_LEVELS];
    const double* fine_forcing; /* scalar fixture fine forcing, n_ff values         */
    int n_ff;
    double eps, length;    /* allen-cahn                                             */
    double newton_tol;
    int newton_max;
    int nx;                /* heat2d: nx*nx interior                                 */
    double cg_rtol;
    int cg_max;
    const double* source;  /* heat2d f (nx*nx) or NULL                               */
    const double* ic;      /* optional initial_condition() override (n values)       */
    /* gray-scott (GrayScott::Options, gray_scott.hpp:24-38); n = 2 nx^2, state
     * [u; v]; newton_tol / newton_max shared with allen-cahn                 */
    double gs_domain, gs_feed, gs_kill, gs_du, gs_dv, gs_linear_tol;
    int gs_reaction, gs_bounds_check;
    double gs_bound_lo, gs_bound_hi;
} atm_problem;

/* Time grid + hierarchy: TimeGrid::make (time_grid.hpp:14-23) and
 * build_hierarchy(fine, m, k) (hierarchy.hpp:84, hierarchy.cpp:24-50). */
typedef struct atm_grid {
    double t0, tf;
    int n_points;
    int n_m;                   /* number of coarsening factors (levels - 1)        */
    int m[ATM_MAX_LEVELS];
    int k;                     /* local-grid distance                              */
} atm_grid;

/* SolverConfig (solver_config.hpp:33-55). */
typedef struct atm_solver {
    int mode, relaxation, nu, max_iters;
    double tol;
    int norm;
    const double* functional_w; /* FunctionalChange, LINEAR: weights w (n values)  */
    int initial_guess;
    uint64_t seed;
    const double* constant_value; /* n values or NULL (=> initial condition)       */
    const double* provided;       /* n_points*n values (InitialGuess::Provided);   *
                                   * copied by atm_setup, unless                    *
                                   * atm_runtime.defer_guess (see there)            */
    int coarse_substeps;
    int functional_kind;          /* atm_functional (FunctionalChange norm only)   */
} atm_solver;

/* Execution / runtime options (replaces SequentialExecution and
 * runtime::ParallelOptions, solver.hpp:138-161, parallel.hpp:13-20). */
typedef struct atm_runtime {
    int device;        /* CUDA device ordinal for this process                     */
    int n_shards;      /* time shards driven by this process (layout.cpp:29-63)    */
    int world_size;    /* >1: one process per GPU, NCCL between processes          */
    int rank;
    const void* nccl_id; /* 128-byte ncclUniqueId (world_size > 1)                 */
    int storage;       /* atm_storage                                              */
    int trace;         /* record per-phase cudaEvent timings                       */
    int reuse_relax;   /* F-relaxation (two-level cycle, and level 0 of FAS V-cycles):
                          skip a cycle's opening level-0 F-sweep, whose results the
                          previous cycle's level-0 correction F-sweep already
                          produced (bitwise the same cycle; opt-in)                */
    int defer_guess;   /* 1: atm_setup sends only the C rows of a provided guess;
                          its F rows are dead under cycling (every cycle rewrites
                          them before reading one) and are copied only if read
                          first (residual norm, level-0 access, kernel entry
                          points, nested init).  The caller's `provided` buffer
                          must then stay valid until the first cycle returns.
                          0 (default): atm_setup copies the whole guess.        */
    int timeout_ms;    /* world_size > 1: an exchange or collective that has not
                          completed after this long aborts the communicator and
                          fails with ATM_RUNTIME_FAULT (ParallelOptions::timeout,
                          parallel.hpp:15; transport.cpp:29-48).  0 = 30000.    */
} atm_runtime;

/* ConvergenceReport (solver_config.hpp:57-64). */
typedef struct atm_report {
    int iterations;
    int converged;
    int stop_reason;   /* 0 converged, 1 max iterations, 2 diverged                */
    double total_seconds;  /* timings["total"]: setup + nested init + iterations   */
    double dof_steps;  /* n x relaxation Phi applications performed (all levels)   */
    double setup_seconds;  /* timings["setup"] (solver.cpp:403-407)                */
} atm_report;

typedef struct atm_ctx atm_ctx;

/* library-level */
int atm_abi_version(void);
const char* atm_create_error(void);          /* message of the last failed create  */
int atm_device_count(void);

/* CycleDriver(app, hier, cfg, ex) + Application::configure
 * (solver.cpp:45-49, application.hpp:50-55). */
atm_status atm_create(const atm_problem* problem, const atm_grid* grid,
                      const atm_solver* solver, const atm_runtime* runtime, atm_ctx** out);
void atm_destroy(atm_ctx* ctx);
const char* atm_last_error(const atm_ctx* ctx);

/* CycleDriver::setup (solver.cpp:81-109) */
atm_status atm_setup(atm_ctx* ctx);
/* CycleDriver::nested_init (solver.cpp:331-368) */
atm_status atm_nested_init(atm_ctx* ctx);
/* CycleDriver::cycle (solver.cpp:322-329) */
atm_status atm_cycle(atm_ctx* ctx);
/* CycleDriver::residual_norm (solver.cpp:370-378) */
atm_status atm_residual_norm(atm_ctx* ctx, double* out);
/* CycleDriver::drive / solve() (solver.cpp:398-435, :485-492): the
 * ConvergenceReport (solver_config.hpp:57-64).  norms[] (residual_norms) and
 * iteration_seconds[] (wall time of each cycle + stopping norm) get one entry
 * per iteration (capacity max_iters); either may be NULL.  Per-phase times
 * (ConvergenceReport::timings) come from atm_phase_times. */
atm_status atm_solve(atm_ctx* ctx, atm_report* report, double* norms, double* iteration_seconds);
/* Fixed-count cycles with one stopping norm each, no host sync in between
 * except the norm readback (bench helper; same arithmetic as atm_solve). */
atm_status atm_iterate(atm_ctx* ctx, int count, double* norms);

/* State access: SpaceTimeState level arrays (space_time.hpp:20-32).
 * which: 0=u 1=g 2=v 3=r.  Host buffers are [count][n]. */
atm_status atm_get_level(atm_ctx* ctx, int level, int which, int first, int count,
                         double* host_out);
atm_status atm_set_level(atm_ctx* ctx, int level, int which, int first, int count,
                         const double* host_in);
int atm_level_points(const atm_ctx* ctx, int level);
int atm_vector_size(const atm_ctx* ctx);
int atm_n_levels(const atm_ctx* ctx);

/* Batched Application::step: out[j] = Phi_{first+j}(in[j]) on `level`
 * (application.hpp:40), and forcing (application.hpp:42-47). */
atm_status atm_apply_phi(atm_ctx* ctx, int level, int first_index, int count,
                         const double* in, double* out);
atm_status atm_forcing(atm_ctx* ctx, int level, int first_index, int count, double* out);

/* kernels:: entry points on the context's device arrays (kernels.hpp:16-67) */
atm_status atm_kernel_f_relax(atm_ctx* ctx, int level, int first_interval, int count);
atm_status atm_kernel_c_relax(atm_ctx* ctx, int level, int first_c, int count);
/* residual r_i for i in [first, first+count) into host_out (kernels.cpp:30-43) */
atm_status atm_kernel_residual(atm_ctx* ctx, int level, int first, int count,
                               double* host_out);

/* Per-phase timings accumulated since creation (PhaseTimer, solver.cpp:11-28;
 * ConvergenceReport::timings): always "setup" and "iterations" (host wall
 * clock); with atm_runtime.trace also the device-event phases "relax",
 * "restrict", "exchange", "coarse", "correct", "norm" (and the level-0 sweep
 * kernels "sweep_relax", "sweep_correct").  Returns the number written (<= cap). */
int atm_phase_times(const atm_ctx* ctx, char* names_csv, int names_cap, double* seconds,
                    int cap);

/* Number of recorded intervals per phase, same order as atm_phase_times. */
int atm_phase_counts(const atm_ctx* ctx, int* counts, int cap);

/* Last-iteration kernel launch count and device time of the dominant kernel
 * (bench helpers). */
atm_status atm_last_iteration_stats(const atm_ctx* ctx, int* launches, double* sweep_ms);

/* Inner linear-solver iterations run since creation (2D heat: CG; Gray-Scott:
 * BiCGSTAB; 0 for the other families) -- the SURVEY 8(d) DOF*CG-iterations
 * unit of the inner-solver configs. */
atm_status atm_inner_iterations(atm_ctx* ctx, unsigned long long* out);

/* Level-0 state bytes moved so far between host and device: the provided
 * guess (atm_setup sends its C rows; its F rows only if something reads them
 * before the first cycle, which rewrites them) and atm_get_level /
 * atm_set_level.  The e2e bench reports these. */
atm_status atm_host_traffic(const atm_ctx* ctx, unsigned long long* h2d, unsigned long long* d2h);

/* `count` cycles + stopping norms, timed on the context's stream with CUDA
 * events (device milliseconds into *device_ms). */
atm_status atm_iterate_timed(atm_ctx* ctx, int count, double* norms, double* device_ms);

/* Page-lock caller-owned host memory for fast host<->device copies. */
atm_status atm_host_register(void* ptr, size_t bytes);
atm_status atm_host_unregister(void* ptr);

/* ---- host-only helpers (no GPU needed) ---------------------------------- */

/* random_state(seed, n) (state_vector.hpp:108-118), host splitmix64 */
void atm_random_state(uint64_t seed, int n, double* out);

/* build_layout (layout.cpp:29-63): per-rank fine/coarsest ownership */
atm_status atm_build_layout(const atm_grid* grid, int workers, int* fine_lo, int* fine_hi,
                            int* coarse_lo, int* coarse_hi);

/* compute_ranges (parallel.cpp:67-130) for one rank: per level
 * [lo, hi] owned points, first/count intervals, first/count C-points,
 * left source / right destination ranks (-1 if none).  Arrays sized L. */
atm_status atm_rank_ranges(const atm_grid* grid, int workers, int rank, int* lo, int* hi,
                           int* iv_first, int* iv_count, int* c_first, int* c_count,
                           int* left_src, int* right_dst);

/* Window payload schedule that replaces the two-round group exchange
 * (parallel.cpp:134-194): rank `rank` needs coarsest indices
 * [need_lo, c_lo-1] from its left; returns the total count of (src_rank,
 * first, count) triples (at most `workers`); min(total, cap) are written to
 * `sends` (capacity cap triples). */
int atm_window_recvs(const atm_grid* grid, int workers, int rank, int* sends, int cap);

/* NCCL unique id for multi-process runs (128 bytes); ATM_RUNTIME_FAULT if
 * NCCL cannot be loaded. */
atm_status atm_nccl_unique_id(void* out128);

#ifdef __cplusplus
}
#endif
#endif /* ATMGRIT_H */
