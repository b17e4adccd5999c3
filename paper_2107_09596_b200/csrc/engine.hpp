// engine.hpp -- host runtime of the B200 AT-MGRIT path.
//
// Replaces the reference's CycleDriver + Execution pair
// (/root/reference/proj/include/tempo/solver.hpp:21-120) with a driver that
// owns device-resident, point-major level arrays per contiguous time shard
// (the rank layout of runtime/layout.hpp:15-40) and drives the Phi kernels.
// Several shards may live in one process on one device ("virtual ranks",
// exchanges are device copies), or one shard per process with NCCL.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "atmgrit.h"
#include "cg_kernels.cuh"
#include "common_kernels.cuh"
#include "heat_kernels.cuh"

struct ncclComm;  // nccl.h: typedef struct ncclComm* ncclComm_t

namespace atm {

struct Error : std::runtime_error {
    atm_status code;
    Error(atm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// ---------------------------------------------------------------------------
// hierarchy and layout (host, no GPU)

struct Hier {
    int L = 0;
    int k = 1;
    double t0 = 0.0;
    std::vector<int> np;    // points per level
    std::vector<int> m;     // coarsening factor per transition
    std::vector<double> dt;
    int coarsest() const { return L - 1; }
    int n_c(int l) const { return (np[l] - 1) / m[l] + 1; }
    // intervals: one after each C-point c with c+1 <= last (hierarchy.cpp:7-22)
    int n_iv(int l) const {
        const int nc = n_c(l);
        return ((nc - 1) * m[l] + 1 <= np[l] - 1) ? nc : nc - 1;
    }
    int stride_total() const {
        int s = 1;
        for (int l = 0; l + 1 < L; ++l) s *= m[l];
        return s;
    }
};

Hier make_hier(const atm_grid& g);

struct Layout {
    int workers = 1;
    std::vector<int> fine_lo, fine_hi, coarse_lo, coarse_hi;
    int owner_of_fine(int i) const;
    int owner_of_coarse(int p) const;
};
Layout build_layout(const Hier& h, int workers);

struct Ranges {
    std::vector<int> lo, hi, iv_first, iv_count, c_first, c_count, left_src, right_dst;
};
Ranges compute_ranges(const Hier& h, const Layout& lay, int rank);

atm_status nccl_unique_id(void* out128);

// ---------------------------------------------------------------------------
// device arrays

struct DArr {
    double* p = nullptr;
    int base = 0;   // global index of row 0
    int rows = 0;
    CUtensorMap tm{};   // one point row per box
    CUtensorMap tmw{};  // one warp slice of a row per box (per-warp stores)
    bool has_tm = false;
    int div = 1;        // > 1: only every div-th point is held (C-point storage)
    bool valid(int i) const {
        return p && i >= base && (i - base) % div == 0 && (i - base) / div < rows;
    }
    // element offset of point i's row
    size_t off(int i, int pitch) const {
        return static_cast<size_t>((i - base) / div) * static_cast<size_t>(pitch);
    }
};

struct LevelDev {
    int lo = 0, hi = -1;
    int iv_first = 0, iv_count = 0, c_first = 0, c_count = 0;
    int left = -1, right = -1;
    int base = 0;     // first allocated global index of every array on this level
    DArr u, g, v, r, w, x;
    bool g_full = false;
    // Phi coefficients
    HeatCoefDev hco{};
    ScalarCoefDev sco{};
    CgCoefDev gco{};
    std::vector<void*> allocs;
};

struct Shard {
    int gid = 0;  // global shard / rank id
    std::vector<LevelDev> lv;
};

struct NcclApi;

class Engine {
public:
    Engine(const atm_problem& p, const atm_grid& g, const atm_solver& s, const atm_runtime& rt);
    ~Engine();

    void setup();
    void nested_init();
    void cycle();
    double residual_norm();            // full level-0 residual (all points)
    double stopping_norm_after_cycle();
    int solve(atm_report* rep, double* norms, double* iteration_seconds = nullptr);
    void iterate(int count, double* norms);

    double iterate_timed(int count, double* norms);  // device ms (CUDA events)
    void xfer_level(int level, int which, int first, int count, double* host, bool to_host);
    void get_level(int level, int which, int first, int count, double* out);
    void set_level(int level, int which, int first, int count, const double* in);
    void apply_phi(int level, int first, int count, const double* in, double* out, bool forcing);
    void kernel_f_relax(int level, int first_iv, int count);
    void kernel_c_relax(int level, int first_c, int count);
    void kernel_residual(int level, int first, int count, double* out);

    int level_points(int l) const { return H_.np[l]; }
    int vector_size() const { return n_; }
    int n_levels() const { return H_.L; }
    int phase_times(char* names, int cap_names, double* secs, int cap, int* counts = nullptr) const;
    int last_launches() const { return last_launches_; }
    double last_sweep_ms() const { return last_sweep_ms_; }
    unsigned long long inner_iterations();
    // state bytes moved between host and device (guess, get/set_level)
    void host_traffic(unsigned long long* h2d, unsigned long long* d2h) const {
        if (h2d) *h2d = h2d_bytes_;
        if (d2h) *d2h = d2h_bytes_;
    }

private:
    // setup helpers
    void alloc_shard(Shard& s);
    void build_coefs(Shard& s);
    // slice_L: chunk length of the sweep kernel that stores into this array
    // by per-warp slices (its slice-map box is 2 slice_L rows)
    DArr alloc_arr(LevelDev& L, int base, int rows, bool tmap, int slice_L = 0);
    void fill_initial_guess();
    void flush_guess();
    void fill_level_rhs(int level);
    // cycle pieces
    // f_dead: the cycle's correction F-sweep rewrites every F row of the
    // level before anything reads it, so only C rows and the rows a later
    // residual / C-relaxation reads are stored (STORE_CF / STORE_NONE)
    void relax_level(int level, bool restrict_tail, bool f_dead);
    void f_sweep(int level, int tail, int store = STORE_ALL);
    void sweep_jobs(Shard& s, int level, int kind, int j0, int j1, int tail, int m_override,
                    double* sq, int sq_base, int store = STORE_ALL);
    void resid_c(int level);  // r at own C (j>=1) of level into level+1 r, plus r_0
    void restrict_to(int level);
    void coarsest_linear();
    void coarsest_fas();
    void correct_from(int level);
    void v_cycle(int level);
    void two_level_cycle();
    void point0_residual(Shard& s, int level, double* r_out, double* sq_out);
    double reduce_norm(double* sq, int count);
    // wait for the stream; with world > 1 a polled wait that fails with
    // ATM_RUNTIME_FAULT on an NCCL async error or after timeout_ms (the
    // communicator is aborted first, transport.cpp:29-61 / parallel.cpp:365-383)
    void sync_stream(const char* what);
    ::ncclComm* comm() const;  // the live communicator (throws after an abort)
    double functional_change();
    // exchanges
    void halo(int level, DArr LevelDev::*arr);
    void window_exchange(int level, DArr LevelDev::*arr);
    void windows(int kind);
    // phi launches
    void window_launch(Shard& s, int level, int kind, int pre_lo, int pre_e0, int pre_e1,
                       int p0, int p1, const DArr& x1, const DArr& x2, const DArr& x3,
                       const DArr& out, int out_stride, int forced, int seed_zero, int idx0,
                       int seed_off);
    int grid_for(int jobs, int occ);
    // timing
    void phase_begin(const char* name);
    void phase_end();
    void check_launch(int err, const char* what);
    void sync_check();

    // configuration
    atm_problem prob_{};
    atm_solver sol_{};
    atm_runtime rt_{};
    Hier H_;
    Layout lay_;
    int n_ = 1, pitch_ = 1, kind_ = 0;
    bool folded_ = false, heat_ = false, ac_ = false, h2d_ = false, gs_ = false;
    bool phi_forced_ = false;
    bool cpts_ = false;      // level-0 u holds only the C points (ATM_STORE_CPOINTS)
    void get_level0_cpts(int first, int count, double* out);
    std::vector<int> Lvl_;   // row-kernel chunk length per level
    int sms_ = 148;
    size_t l2_bytes_ = 0;  // device L2 size: rows of arrays well past it are stored evict_first
    int world_ = 1, rank_ = 0, G_ = 1;
    std::vector<double> ic_, ff_, fw_, cval_, prov_, src_;
    double h_ = 0.0;
    std::vector<double> sinp_;
    std::vector<Shard> sh_;
    std::vector<Ranges> ranges_all_;  // compute_ranges of every rank (exchange schedules)
    int timeout_ms_ = 30000;
    cudaStream_t st_ = nullptr;
    bool setup_done_ = false;
    // global reduction arrays (per point of level 0)
    double* d_sq_full_ = nullptr;
    double* d_sq_c_ = nullptr;
    double* d_sq_all_ = nullptr;  // world > 1: all-reduced per-point squares
    double* d_norm_ = nullptr;
    double* d_prevf_ = nullptr;
    double* d_fmax_ = nullptr;
    double* d_fw_ = nullptr;
    double* d_ic_ = nullptr;
    double* d_row_ = nullptr;
    double* d_ff_ = nullptr;
    double* d_prof_ = nullptr;
    int* d_fail_ = nullptr;   // Allen-Cahn Newton / heat2d CG failure flag
    unsigned long long* d_inner_ = nullptr;  // inner CG / BiCGSTAB iterations run so far
    double* d_src_ = nullptr; // heat2d source f
    int cl_ = 1;              // heat1d rows split over a cluster of cl_ CTAs (n > 5376)
    double* d_xg_ = nullptr;  // heat2d CG x scratch (one row per resident cluster)
    double* d_gex_ = nullptr;  // heat2d CG group mode: exchange rows / partials per group
    unsigned long long* d_gflag_ = nullptr;  // heat2d CG group mode: per-CTA sequence flags
    void check_newton();
    std::vector<void*> gallocs_;
    // NCCL (world > 1)
    std::unique_ptr<NcclApi> nccl_;
    void* comm_ = nullptr;
    // timing (ConvergenceReport::timings: host "setup" / "iterations" always,
    // device-event phases with trace_)
    void host_phase(const char* name, double seconds);
    bool trace_ = false;
    std::map<std::string, double> phase_sec_;
    struct Pending : std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>> {
        bool closed = false;
    };
    std::vector<Pending> pending_;
    std::map<std::string, int> phase_cnt_;
    const double* prov_ptr_ = nullptr;
    // level-0 F rows of a provided guess not yet copied (setup sent the C
    // rows only; the first cycle overwrites every F row before reading it)
    bool guess_pending_ = false;
    unsigned long long h2d_bytes_ = 0, d2h_bytes_ = 0;
    const char* cur_phase_ = nullptr;
    cudaEvent_t cur_ev_ = nullptr;
    std::vector<cudaEvent_t> ev_pool_;
    int launches_ = 0, last_launches_ = 0;
    // CUDA graph of one cycle (captured on the first cycle, then replayed)
    bool use_graphs() const;
    bool reuse_possible() const;
    bool relax_valid_ = false;  // level-1 r holds the residuals of the current C points
    // multi-process two-level F cycles: the level-0 left-edge row still holds
    // the left neighbour's current last C point (nothing has written a C point
    // since the correction sweep's exchange), so the next cycle's opening
    // F-sweep needs no second halo exchange
    bool halo0_valid_ = false;
    cudaGraphExec_t graph_exec_ = nullptr;
    int graph_launches_ = 0;
    double last_sweep_ms_ = 0.0;
};

}  // namespace atm
