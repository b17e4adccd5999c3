// engine.cpp -- host runtime of the B200 AT-MGRIT path (see engine.hpp).
//
// Reference citations are relative to /root/reference/proj.
#include "engine.hpp"

#include <cstdio>

#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <sstream>
#include <thread>

namespace atm {

namespace {

constexpr double kPi = 3.14159265358979323846;

[[noreturn]] void config_error(const std::string& m) { throw Error(ATM_CONFIG_ERROR, m); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(ATM_RUNTIME_FAULT, std::string("CUDA error: ") + cudaGetErrorString(e) +
                                           " in " + what);
}
#define CK(x) ck((x), #x)

int ceil_div(int a, int b) { return (a + b - 1) / b; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            throw Error(ATM_RUNTIME_FAULT, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2D view [rows * pitch/16][16 doubles], box = one point row, 128B swizzle.
CUtensorMap make_row_map(double* ptr, int rows, int pitch) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t dims[2] = {16, static_cast<cuuint64_t>(rows) * (pitch / 16)};
    const cuuint64_t strides[1] = {128};
    // a box holds at most 256 rows of the view: longer point rows (pitch a
    // multiple of 256) are moved as two half-row boxes (tma_load_row), rows
    // split over a cluster (pitch a multiple of 4096 past 8192) as one box per
    // CTA part
    const int R = pitch / 16;
    const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(R <= 256 ? R : R <= 512 ? R / 2 : 256)};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ptr, dims, strides, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(ATM_RUNTIME_FAULT, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

// 3D view [rows][pitch/16][16 doubles], box = one warp's slice of a row
// (32 threads x L doubles = 2L lines of 128 B), 128B swizzle; the part of a
// box past the row end is clipped by the TMA unit.
CUtensorMap make_slice_map(double* ptr, int rows, int pitch, int L) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(pitch / 16), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(pitch) * 8};
    const cuuint32_t box[3] = {16, static_cast<cuuint32_t>(std::min(2 * L, pitch / 16)), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ptr, dims, strides, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(ATM_RUNTIME_FAULT, "cuTensorMapEncodeTiled (slice) failed (" + std::to_string(r) + ")");
    return m;
}

}  // namespace

// ---------------------------------------------------------------------------
// NCCL, loaded lazily so the library has no link-time NCCL dependency

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*ErrStr)(ncclResult_t) = nullptr;
    // fault detection (optional symbols: a stand-in may lack them)
    ncclResult_t (*GetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Abort)(ncclComm_t) = nullptr;

    bool load() {
        if (h) return true;
        // ATM_NCCL_LIB: an alternative implementation of the same entry
        // points (tests/mocknccl: host-mediated transport for several
        // processes on one GPU)
        if (const char* alt = std::getenv("ATM_NCCL_LIB")) h = dlopen(alt, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
#define SYM(f, n) f = reinterpret_cast<decltype(f)>(dlsym(h, n)); if (!f) return false
        SYM(GetUniqueId, "ncclGetUniqueId");
        SYM(CommInitRank, "ncclCommInitRank");
        SYM(CommDestroy, "ncclCommDestroy");
        SYM(Send, "ncclSend");
        SYM(Recv, "ncclRecv");
        SYM(GroupStart, "ncclGroupStart");
        SYM(GroupEnd, "ncclGroupEnd");
        SYM(AllReduce, "ncclAllReduce");
        SYM(ErrStr, "ncclGetErrorString");
#undef SYM
        GetAsyncError = reinterpret_cast<decltype(GetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
        Abort = reinterpret_cast<decltype(Abort)>(dlsym(h, "ncclCommAbort"));
        return true;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw Error(ATM_RUNTIME_FAULT, std::string("NCCL error in ") + what + ": " + ErrStr(r));
    }
};

static NcclApi& nccl_global() {
    static NcclApi api;
    return api;
}

atm_status nccl_unique_id(void* out) {
    NcclApi& api = nccl_global();
    if (!api.load()) return ATM_RUNTIME_FAULT;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return ATM_RUNTIME_FAULT;
    std::memcpy(out, &id, sizeof(id));
    return ATM_OK;
}

// ---------------------------------------------------------------------------
// hierarchy / layout / ranges (host restatements)

Hier make_hier(const atm_grid& g) {
    // TimeGrid::make (time_grid.hpp:14-23)
    if (g.n_points < 2) config_error("TimeGrid: need at least 2 points");
    if (!(g.tf > g.t0)) config_error("TimeGrid: tf must exceed t0");
    // build_hierarchy (hierarchy.cpp:24-50)
    if (g.n_m < 1 || g.n_m >= ATM_MAX_LEVELS) config_error("hierarchy needs at least one coarsening factor");
    if (g.k < 1) config_error("local-grid distance k must be at least 1");
    Hier h;
    h.L = g.n_m + 1;
    h.k = g.k;
    h.t0 = g.t0;
    h.np.push_back(g.n_points);
    h.dt.push_back((g.tf - g.t0) / static_cast<double>(g.n_points - 1));
    for (int l = 0; l < g.n_m; ++l) {
        if (g.m[l] < 2) config_error("coarsening factor must exceed 1, got " + std::to_string(g.m[l]));
        const int nc = (h.np.back() - 1) / g.m[l] + 1;
        if (nc < 2)
            config_error("coarsening exhausts the grid at level " + std::to_string(l + 1) + " (" +
                         std::to_string(nc) + " points)");
        h.m.push_back(g.m[l]);
        h.np.push_back(nc);
        h.dt.push_back(h.dt.back() * g.m[l]);
    }
    return h;
}

int Layout::owner_of_fine(int i) const {
    for (int r = 0; r < workers; ++r)
        if (i >= fine_lo[r] && i <= fine_hi[r]) return r;
    config_error("layout: fine point " + std::to_string(i) + " is unowned");
}

int Layout::owner_of_coarse(int p) const {
    for (int r = 0; r < workers; ++r)
        if (p >= coarse_lo[r] && p <= coarse_hi[r]) return r;
    config_error("layout: coarse point " + std::to_string(p) + " is unowned");
}

// layout.cpp:29-63: near-even split of coarsest C-points; fine block
// (T_{lo-1}, T_hi], point 0 with the first rank, trailing points with the last.
Layout build_layout(const Hier& h, int workers) {
    const int n_coarse = h.np.back();
    if (workers < 1) config_error("layout: need at least one worker");
    if (workers > n_coarse)
        config_error("layout: " + std::to_string(workers) + " workers exceed the " +
                     std::to_string(n_coarse) + " coarsest-level points");
    const int stride = h.stride_total();
    const int n_fine = h.np[0];
    Layout lay;
    lay.workers = workers;
    const int base = n_coarse / workers, extra = n_coarse % workers;
    int next = 0;
    for (int r = 0; r < workers; ++r) {
        const int size = base + (r < extra ? 1 : 0);
        const int lo = next, hi = next + size - 1;
        next = hi + 1;
        lay.coarse_lo.push_back(lo);
        lay.coarse_hi.push_back(hi);
        lay.fine_lo.push_back(r == 0 ? 0 : (lo - 1) * stride + 1);
        lay.fine_hi.push_back(r == workers - 1 ? n_fine - 1 : hi * stride);
    }
    return lay;
}

// parallel.cpp:67-130
Ranges compute_ranges(const Hier& h, const Layout& lay, int rank) {
    const int L = h.L;
    Ranges rr;
    rr.lo.assign(L, 0);
    rr.hi.assign(L, -1);
    rr.iv_first.assign(L, 0);
    rr.iv_count.assign(L, 0);
    rr.c_first.assign(L, 0);
    rr.c_count.assign(L, 0);
    rr.left_src.assign(L, -1);
    rr.right_dst.assign(L, -1);
    const int fine_lo = lay.fine_lo[rank], fine_hi = lay.fine_hi[rank];
    int stride = 1;
    for (int l = 0; l < L; ++l) {
        const int n_l = h.np[l];
        const int lo = ceil_div(fine_lo, stride);
        const int hi = std::min(fine_hi / stride, n_l - 1);
        rr.lo[l] = lo;
        rr.hi[l] = hi;
        const bool empty = lo > hi;
        if (!empty) {
            if (lo > 0) rr.left_src[l] = lay.owner_of_fine((lo - 1) * stride);
            if (hi + 1 <= n_l - 1) rr.right_dst[l] = lay.owner_of_fine((hi + 1) * stride);
        }
        if (l < L - 1) {
            const int m = h.m[l];
            if (!empty) {
                const int cf = ceil_div(lo, m), cl = hi / m;
                if (cf <= cl) {
                    rr.c_first[l] = cf;
                    rr.c_count[l] = cl - cf + 1;
                }
                // intervals whose first F-point lies in [lo, hi]
                const int niv = h.n_iv(l);
                int first = -1, count = 0;
                for (int nI = std::max(0, (lo - 1) / m - 1); nI < niv; ++nI) {
                    const int f = nI * m + 1;
                    if (f > hi) break;
                    if (f >= lo) {
                        if (first < 0) first = nI;
                        ++count;
                    }
                }
                rr.iv_first[l] = count > 0 ? first : 0;
                rr.iv_count[l] = count;
            }
            stride *= m;
        }
    }
    return rr;
}

// ---------------------------------------------------------------------------
// Engine: construction

Engine::Engine(const atm_problem& p, const atm_grid& g, const atm_solver& s, const atm_runtime& rt)
    : prob_(p), sol_(s), rt_(rt) {
    H_ = make_hier(g);
    if (s.coarse_substeps < 1) config_error("coarse_substeps must be at least 1");
    kind_ = p.kind;
    switch (kind_) {
        case ATM_PHI_HEAT1D:
            n_ = p.n;
            if (n_ < 1) config_error("heat1d: need at least one spatial unknown");
            if (!(p.x1 > p.x0)) config_error("heat1d: x1 must exceed x0");
            // one CTA holds one state vector up to n = 5376 (the FAS window
            // kernel stages five rows, 5 x 42 KB of the 227 KB); past that a
            // row is split over a cluster of up to 8 CTAs of 4096 elements
            if (n_ > kMaxCluster * 4096)
                config_error("heat1d: n > " + std::to_string(kMaxCluster * 4096) +
                             " exceeds a cluster of " + std::to_string(kMaxCluster) + " row CTAs");
            if (n_ > 5376) cl_ = (n_ + 4095) / 4096;
            heat_ = true;
            folded_ = p.folded != 0;
            break;
        case ATM_PHI_DAHLQUIST:
        case ATM_PHI_SCALAR:
            n_ = 1;
            folded_ = p.folded != 0;
            if (kind_ == ATM_PHI_SCALAR && p.n_mult < H_.L)
                config_error("scalar: one multiplier per level");
            break;
        case ATM_PHI_ALLEN_CAHN:
            // BASELINE config 3 (no reference Phi; oracle/atm_oracle.c ac_step)
            n_ = p.n;
            if (n_ < 16 || n_ > 4096) config_error("allen-cahn: n must be in [16, 4096]");
            if (!(p.eps > 0.0) || !(p.length > 0.0)) config_error("allen-cahn: bad eps/length");
            if (!(p.newton_tol > 0.0) || p.newton_max < 1)
                config_error("allen-cahn: newton_tol > 0 and newton_max >= 1 required");
            heat_ = true;  // row kernels
            ac_ = true;
            folded_ = true;
            break;
        case ATM_PHI_GRAY_SCOTT:
            // problems::GrayScott (gray_scott.cpp:16-190): runs on the cluster
            // CG machinery with a single-CTA Newton + BiCGSTAB Phi
            if (p.nx < 4) config_error("gray-scott: grid must be at least 4x4");
            if (!(p.gs_domain > 0.0)) config_error("gray-scott: domain size must be positive");
            if (!(p.newton_tol > 0.0) || p.newton_max < 1 || !(p.gs_linear_tol > 0.0))
                config_error("gray-scott: newton_tol, linear_tol > 0 and newton_max >= 1 required");
            n_ = 2 * p.nx * p.nx;
            h2d_ = true;
            gs_ = true;
            folded_ = true;
            break;
        case ATM_PHI_HEAT2D:
            // BASELINE configs 2, 4 (no reference Phi; oracle/atm_oracle.c h2_solve)
            if (p.nx < 1) config_error("heat2d: need at least one interior point per side");
            if (p.nx > 1024) config_error("heat2d: nx > 1024 exceeds the cluster CG kernel");
            if (!(p.cg_rtol > 0.0) || p.cg_max < 1)
                config_error("heat2d: cg_rtol > 0 and cg_max >= 1 required");
            n_ = p.nx * p.nx;
            h2d_ = true;
            folded_ = p.folded != 0;
            break;
        default:
            config_error("unknown problem kind " + std::to_string(kind_));
    }
    // CycleDriver::validate (solver.cpp:51-79)
    if (!(s.tol > 0.0)) config_error("solver: tol must be positive");
    if (s.max_iters < 1) config_error("solver: max_iters must be at least 1");
    if (s.relaxation == ATM_RELAX_FCF && s.nu < 1) config_error("solver: FCF relaxation needs nu >= 1");
    if (s.mode == ATM_TWO_LEVEL) {
        if (H_.L != 2) config_error("two-level mode needs a two-level hierarchy");
        if (folded_) config_error("two-level residual-correction mode needs explicit forcing");
    } else if (!folded_) {
        config_error("FAS cycles need forcing folded into the integrator");
    }
    if (s.norm == ATM_NORM_FUNCTIONAL) {
        if (s.functional_kind != ATM_FUNCTIONAL_LINEAR && s.functional_kind != ATM_FUNCTIONAL_NORM2)
            config_error("functional-change stopping norm: unknown functional");
        if (s.functional_kind == ATM_FUNCTIONAL_LINEAR && !s.functional_w)
            config_error("functional-change stopping norm needs a functional");
    }
    if (s.initial_guess == ATM_GUESS_PROVIDED && !s.provided)
        config_error("provided initial guess has the wrong number of points");
    // C-point storage (atm_storage): level 0 keeps only its
    // C points; F values are the F-relaxation of their interval's C point
    // (recomputed on read).  Every level-0 F row must then be a pure function
    // of the C rows: F-relaxation only, and no stored level-0 forcing.
    if (rt.storage != ATM_STORE_FULL && rt.storage != ATM_STORE_CPOINTS)
        config_error("runtime: unknown storage mode");
    if (rt.storage == ATM_STORE_CPOINTS) {
        if (H_.L < 2) config_error("C-point storage needs at least two levels");
        if (s.relaxation != ATM_RELAX_F) config_error("C-point storage needs F-relaxation");
        const bool g0_full = !folded_ && ((heat_ && !ac_ && p.manufactured) ||
                                          (h2d_ && !gs_ && p.source) ||
                                          (kind_ == ATM_PHI_SCALAR && p.fine_forcing && p.n_ff > 0));
        if (g0_full) config_error("C-point storage needs the forcing folded into Phi");
        cpts_ = true;
    }

    pitch_ = (heat_ || h2d_) ? ((n_ + 15) / 16) * 16 : 1;
    // L = 32 row kernels (pitch > 2048): a thread's chunk must not straddle
    // the row end, so rows are whole 32-element chunks
    if (heat_ && !ac_ && pitch_ > 2048) pitch_ = ((n_ + 31) / 32) * 32;
    // 4096 < n <= 5376: a point row is loaded / stored as two TMA boxes of
    // half a row each (a box holds at most 256 rows of the [.., 16] view, and
    // a 128B-swizzled box must start 1024-byte aligned), so the row is padded
    // to a multiple of 256 (padding stays 0)
    if (heat_ && !ac_ && pitch_ > 4096) pitch_ = ((n_ + 255) / 256) * 256;
    // rows split over a cluster: CTA q holds elements [4096 q, 4096 q + 4096)
    if (cl_ > 1) pitch_ = 4096 * cl_;
    // host copies of caller-owned inputs
    ic_.assign(n_, 0.0);
    if (heat_ && !ac_) {
        h_ = (p.x1 - p.x0) / static_cast<double>(n_ + 1);  // heat1d.cpp:16
        sinp_.resize(n_);
        for (int i = 0; i < n_; ++i) sinp_[i] = std::sin(kPi * (p.x0 + h_ * (i + 1)));
        ic_ = sinp_;  // heat1d.cpp:85-91
    } else if (!ac_ && !h2d_) {
        ic_[0] = p.u0;
    }
    if (h2d_ && !gs_ && p.source) src_.assign(p.source, p.source + n_);
    if (gs_) {
        // GrayScott::initial_condition (gray_scott.cpp:38-61): u = 1, v = 0
        // plus the sin^2 bump on [1, 1.5]^2, cell centres (j + 1/2) h
        const int nx = p.nx, cells = nx * nx;
        const double h = p.gs_domain / nx;
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < nx; ++j) {
                const int c = i * nx + j;
                const double x = (j + 0.5) * h, y = (i + 0.5) * h;
                double u = 1.0, v = 0.0;
                if (x >= 1.0 && x <= 1.5 && y >= 1.0 && y <= 1.5) {
                    const double sx = std::sin(4.0 * kPi * x), sy = std::sin(4.0 * kPi * y);
                    const double bump = 0.25 * sx * sx * sy * sy;
                    u = 1.0 - 2.0 * bump;
                    v = bump;
                }
                ic_[c] = u;
                ic_[cells + c] = v;
            }
        if (p.ic) ic_.assign(p.ic, p.ic + n_);
    }
    if (p.ic) ic_.assign(p.ic, p.ic + n_);
    if (kind_ == ATM_PHI_SCALAR && p.fine_forcing && p.n_ff > 0)
        ff_.assign(p.fine_forcing, p.fine_forcing + p.n_ff);
    if (s.functional_w && s.functional_kind == ATM_FUNCTIONAL_LINEAR)
        fw_.assign(s.functional_w, s.functional_w + n_);
    if (s.constant_value) cval_.assign(s.constant_value, s.constant_value + n_);
    // the provided guess stays caller-owned until the first cycle (no host copy:
    // it can be the full level-0 array)
    prov_ptr_ = s.provided;
    prob_.ic = nullptr;
    prob_.fine_forcing = nullptr;
    prob_.source = nullptr;
    sol_.functional_w = nullptr;
    sol_.constant_value = nullptr;
    sol_.provided = nullptr;

    world_ = std::max(1, rt.world_size);
    rank_ = rt.rank;
    const int local = std::max(1, rt.n_shards);
    if (world_ > 1 && local != 1) config_error("multi-process runs drive one shard per process");
    G_ = world_ > 1 ? world_ : local;
    lay_ = build_layout(H_, G_);
    for (int q = 0; q < G_; ++q) ranges_all_.push_back(compute_ranges(H_, lay_, q));
    if (rt.timeout_ms < 0) config_error("runtime: timeout_ms must be >= 0");
    if (rt.timeout_ms > 0) timeout_ms_ = rt.timeout_ms;
    trace_ = rt.trace != 0;
    // chunk length per level: n > 2048 sweeps run 128-thread CTAs (L = 32,
    // three per SM); the coarsest level (windows only) keeps 256 threads
    // (L = 16), whose window kernel holds twice the warps per SM
    Lvl_.assign(H_.L, 16);
    for (int l = 0; l < H_.L; ++l) {
        int L = 2;
        while (L < 16 && pitch_ / L > 256) L *= 2;
        // (ATM_WIN_L32: also the coarsest level -- measured slower, 0.79 vs 0.72 ms)
        if (pitch_ > 2048 && (l < H_.coarsest() || std::getenv("ATM_WIN_L32"))) L = 32;
        if (const char* e = std::getenv("ATM_HEAT_L")) L = std::atoi(e);
        if (ac_) L = 8;
        if (cl_ > 1) L = 32;  // cluster rows: 128 threads x 32 elements per CTA part
        Lvl_[l] = L;
    }

    CK(cudaSetDevice(rt.device));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
    {
        int l2 = 0;
        CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
        l2_bytes_ = static_cast<size_t>(std::max(l2, 0));
    }
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));

    if (world_ > 1) {
        nccl_.reset(new NcclApi());
        if (!nccl_->load()) throw Error(ATM_RUNTIME_FAULT, "cannot load libnccl.so.2");
        if (!rt.nccl_id) config_error("multi-process run needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, rt.nccl_id, sizeof(id));
        ncclComm_t c = nullptr;
        nccl_->check(nccl_->CommInitRank(&c, world_, id, rank_), "ncclCommInitRank");
        comm_ = c;
    }

    // shards driven by this process
    if (world_ > 1) {
        sh_.resize(1);
        sh_[0].gid = rank_;
    } else {
        sh_.resize(G_);
        for (int i = 0; i < G_; ++i) sh_[i].gid = i;
    }
    // global buffers
    auto dalloc = [&](size_t bytes) {
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        CK(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
        gallocs_.push_back(p);
        return static_cast<double*>(p);
    };
    const int np0 = H_.np[0];
    // stopping-norm squares: one per level-0 C point (F residuals are zero
    // after a cycle); the full residual norm keeps one per point
    const int nc0 = H_.n_c(0);
    d_sq_full_ = dalloc(sizeof(double) * np0);
    d_sq_c_ = dalloc(sizeof(double) * nc0);
    if (world_ > 1) d_sq_all_ = dalloc(sizeof(double) * std::max(np0, nc0));
    d_norm_ = dalloc(sizeof(double) * 300);
    d_fmax_ = dalloc(sizeof(double) * std::max(1, G_));
    d_prevf_ = dalloc(sizeof(double) * nc0);
    d_ic_ = dalloc(sizeof(double) * pitch_);
    d_row_ = dalloc(sizeof(double) * pitch_);
    d_fail_ = reinterpret_cast<int*>(dalloc(sizeof(int) * 4));
    d_inner_ = reinterpret_cast<unsigned long long*>(dalloc(sizeof(unsigned long long)));
    if (!src_.empty()) {
        d_src_ = dalloc(sizeof(double) * n_);
        CK(cudaMemcpy(d_src_, src_.data(), sizeof(double) * n_, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(d_ic_, ic_.data(), sizeof(double) * n_, cudaMemcpyHostToDevice));
    if (!fw_.empty()) {
        d_fw_ = dalloc(sizeof(double) * n_);
        CK(cudaMemcpy(d_fw_, fw_.data(), sizeof(double) * n_, cudaMemcpyHostToDevice));
    }
    if (!ff_.empty()) {
        d_ff_ = dalloc(sizeof(double) * ff_.size());
        CK(cudaMemcpy(d_ff_, ff_.data(), sizeof(double) * ff_.size(), cudaMemcpyHostToDevice));
    }
    // Phi adds its forcing itself (folded integrators with a source term)
    phi_forced_ = folded_ && ((heat_ && !ac_ && prob_.manufactured) || (h2d_ && d_src_));
    for (Shard& s : sh_) alloc_shard(s);
    for (Shard& s : sh_) build_coefs(s);
}

Engine::~Engine() {
    if (st_) cudaStreamSynchronize(st_);
    for (Shard& s : sh_)
        for (LevelDev& L : s.lv)
            for (void* p : L.allocs) cudaFree(p);
    for (void* p : gallocs_) cudaFree(p);
    for (auto& pe : pending_) {
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (comm_ && nccl_) nccl_->CommDestroy(static_cast<ncclComm_t>(comm_));
    if (st_) cudaStreamDestroy(st_);
}

DArr Engine::alloc_arr(LevelDev& L, int base, int rows, bool tmap, int slice_L) {
    DArr a;
    a.base = base;
    a.rows = std::max(rows, 0);
    if (a.rows == 0) return a;
    const size_t bytes = sizeof(double) * static_cast<size_t>(a.rows) * pitch_;
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMemsetAsync(p, 0, bytes, st_));
    L.allocs.push_back(p);
    a.p = static_cast<double*>(p);
    if (tmap && heat_) {
        a.tm = make_row_map(a.p, a.rows, pitch_);
        a.tmw = make_slice_map(a.p, a.rows, pitch_, slice_L > 0 ? slice_L : 16);
        a.has_tm = true;
    }
    return a;
}

void Engine::alloc_shard(Shard& s) {
    const Ranges rr = compute_ranges(H_, lay_, s.gid);
    const int L = H_.L, lc = H_.coarsest();
    s.lv.resize(L);
    for (int l = 0; l < L; ++l) {
        LevelDev& Lv = s.lv[l];
        Lv.lo = rr.lo[l];
        Lv.hi = rr.hi[l];
        Lv.iv_first = rr.iv_first[l];
        Lv.iv_count = rr.iv_count[l];
        Lv.c_first = rr.c_first[l];
        Lv.c_count = rr.c_count[l];
        Lv.left = rr.left_src[l];
        Lv.right = rr.right_dst[l];
        if (Lv.hi < Lv.lo) continue;
        int base = std::max(0, Lv.lo - 1);
        if (l == lc && l >= 1) base = std::min(base, std::max(0, Lv.lo - H_.k + 1));
        Lv.base = base;
        const int rows = Lv.hi - base + 1;
        if (l == 0 && cpts_) {
            // base (0 or the left shard's last point) is a C point
            const int m0 = H_.m[0];
            Lv.u = alloc_arr(Lv, base, Lv.hi / m0 - base / m0 + 1, true, Lvl_.empty() ? 0 : Lvl_[l]);
            Lv.u.div = m0;
        } else {
            Lv.u = alloc_arr(Lv, base, rows, true, Lvl_.empty() ? 0 : Lvl_[l]);
        }
        // g: full per-point array where forcing is stored, else point 0 only
        bool g_full = false;
        if (l == 0 && !folded_) {
            const bool heat_forced = (heat_ && !ac_ && prob_.manufactured) || (h2d_ && d_src_);
            const bool scalar_forced = (kind_ == ATM_PHI_SCALAR) && !ff_.empty();
            g_full = heat_forced || scalar_forced;
        }
        if (l >= 1 && l < lc && sol_.mode != ATM_TWO_LEVEL) g_full = true;
        Lv.g_full = g_full;
        if (g_full) Lv.g = alloc_arr(Lv, base, rows, true);
        else if (base == 0) Lv.g = alloc_arr(Lv, 0, 1, true);
        if (l >= 1) {
            Lv.v = alloc_arr(Lv, base, rows, true);
            Lv.r = alloc_arr(Lv, base, rows, true, Lvl_.empty() ? 0 : Lvl_[l - 1]);
            if (l == lc && sol_.mode != ATM_TWO_LEVEL) {
                Lv.w = alloc_arr(Lv, base, rows, true);
                Lv.x = alloc_arr(Lv, base, rows, true);
            }
        }
    }
}

void Engine::build_coefs(Shard& s) {
    const int L = H_.L, lc = H_.coarsest();
    for (int l = 0; l < L; ++l) {
        LevelDev& Lv = s.lv[l];
        const int S = (l == lc) ? sol_.coarse_substeps : 1;  // solver.cpp:39
        const double dt = H_.dt[l];
        const double sub_dt = dt / S;
        auto up = [&](const std::vector<double>& v) {
            void* p = nullptr;
            CK(cudaMalloc(&p, sizeof(double) * std::max<size_t>(v.size(), 1)));
            if (!v.empty())
                CK(cudaMemcpy(p, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice));
            Lv.allocs.push_back(p);
            return static_cast<const double*>(p);
        };
        if (heat_) {
            // Allen-Cahn: the Newton inner solve uses the shifted linear part
            // A_s = tridiag(-dt c, 1 + 2 dt c - dt + s, -dt c), cyclic
            const double ac_c = ac_ ? prob_.eps * prob_.eps /
                                          ((prob_.length / n_) * (prob_.length / n_))
                                    : 0.0;
            const double ac_s = 1.5 * sub_dt;
            HeatLevelHost hh =
                ac_ ? heat_level_host(n_, pitch_, Lvl_[l], sub_dt * ac_c, ac_s - sub_dt, S, true)
                : cl_ > 1 ? heat_cluster_host(n_, cl_, sub_dt / (h_ * h_), S)
                          : heat_level_host(n_, pitch_, Lvl_[l], sub_dt / (h_ * h_), 0.0, S, false);
            HeatCoefDev& c = Lv.hco;
            c.cl = cl_;
            c.blk = c.cS = nullptr;
            if (cl_ > 1) {
                c.blk = up(hh.blk);
                c.cS = up(hh.cS);
            }
            c.xw = up(hh.xw);
            c.cyclic = hh.cyclic;
            c.ncw_r0 = hh.ncw_r0;
            c.tl = hh.tl;
            c.pl = hh.pl;
            for (int q = 0; q < 4; ++q) c.S[q] = hh.S[q];
            c.ql = hh.ql;
            c.pbl = hh.pbl;
            c.prob = ac_ ? 1 : 0;
            if (ac_) {
                c.ac_dt = sub_dt;
                c.ac_c = ac_c;
                c.ac_shift = ac_s;
                c.newton_tol = prob_.newton_tol;
                c.newton_max = prob_.newton_max;
                c.ac_umax2 = 1.0;
                c.inner_eta = 1e-15;
                c.fail = d_fail_;
            }
            if (!(hh.fit_err <= 1e-13))
                throw Error(ATM_RUNTIME_FAULT, "heat Phi: boundary-correction carries do not "
                                               "reproduce w (rel err " +
                                                   std::to_string(hh.fit_err) + ")");
            c.scan = up(hh.scan);
            c.wf = up(hh.wf);
            c.wb = up(hh.wb);
            c.wk = up(hh.wk);
            c.powc = up(hh.powc);
            c.beta_c = hh.beta_c;
            c.gamma_c = hh.gamma_c;
            c.cneg_c = hh.cneg_c;
            c.sigma = hh.sigma;
            c.ncw = hh.ncw;
            c.sb_m = hh.sb_m;
            c.sb_af = hh.sb_af;
            c.sb_ab = hh.sb_ab;
            for (int e = 0; e < 8; ++e) {
                c.sb_q[e] = hh.sb_q[e];
                c.sb_pb[e] = hh.sb_pb[e];
            }
            c.n = n_;
            c.pitch = pitch_;
            c.nt = hh.nt;
            c.L = hh.L;
            c.substeps = S;
            if (prob_.manufactured && !ac_) {
                // theta per (index, substep): heat1d.cpp:72-75 evaluated on the host
                const int np = H_.np[l];
                std::vector<double> th(static_cast<size_t>(np) * S, 0.0);
                for (int i = 1; i < np; ++i)
                    for (int ss = 1; ss <= S; ++ss) {
                        const double t = (H_.t0 + dt * (i - 1)) + sub_dt * ss;
                        th[static_cast<size_t>(i) * S + (ss - 1)] =
                            sub_dt * (-(std::sin(t) - kPi * kPi * std::cos(t)));
                    }
                c.theta = up(th);
                std::vector<double> prof(std::max(static_cast<size_t>(hh.nt) * hh.L, static_cast<size_t>(pitch_)), 0.0);
                for (int i = 0; i < n_; ++i) prof[i] = sinp_[i];
                c.prof = up(prof);
            }
        } else if (gs_) {
            CgCoefDev& c = Lv.gco;
            c.pitch = pitch_;
            // with the work vectors in global scratch, a level with few
            // concurrent systems (intervals, or windows on the coarsest level)
            // gives each Phi a cluster of several CTAs
            const int jobs = (l == H_.coarsest()) ? H_.np[l] : std::max(1, H_.n_iv(l));
            int cs = 1;
            while (cs < 8 && jobs * cs * 2 <= sms_) cs *= 2;
            if (const char* e = std::getenv("ATM_GS_CS")) cs = std::atoi(e);
            if (!gs_geometry(prob_.nx, c, cs)) config_error("gray-scott: unsupported grid");
            if (!c.x_smem) {
                // ten work vectors per resident cluster in global scratch
                // (per level: the cluster size, hence the slot count, differs)
                const int ncl = cg_max_clusters(c);
                void* p = nullptr;
                CK(cudaMalloc(&p, sizeof(double) * 10 * static_cast<size_t>(ncl) * pitch_));
                Lv.allocs.push_back(p);
                c.xg = static_cast<double*>(p);
            }
            const double h = prob_.gs_domain / prob_.nx;
            c.gs_h2inv = 1.0 / (h * h);
            c.gs_du = prob_.gs_du;
            c.gs_dv = prob_.gs_dv;
            c.gs_feed = prob_.gs_feed;
            c.gs_kill = prob_.gs_kill;
            c.gs_linear_tol = prob_.gs_linear_tol;
            c.gs_reaction = prob_.gs_reaction;
            c.gs_bounds_check = prob_.gs_bounds_check;
            c.gs_bound_lo = prob_.gs_bound_lo;
            c.gs_bound_hi = prob_.gs_bound_hi;
            c.newton_tol = prob_.newton_tol;
            c.newton_max = prob_.newton_max;
            c.sdt = sub_dt;
            c.substeps = S;
            c.fail = d_fail_;
            c.iters = d_inner_;
        } else if (h2d_) {
            CgCoefDev& c = Lv.gco;
            c.pitch = pitch_;
            cg_geometry(prob_.nx, c);
            if (c.cs < 1) config_error("heat2d: nx too large for the cluster CG kernel");
            const double hh = 1.0 / static_cast<double>(prob_.nx + 1);
            c.c = sub_dt / (hh * hh);
            c.diag = 1.0 + 4.0 * c.c;
            c.sdt = sub_dt;
            c.src = d_src_;
            c.substeps = S;
            c.rtol = prob_.cg_rtol;
            c.cg_max = prob_.cg_max;
            c.fail = d_fail_;
            c.iters = d_inner_;
            if (!c.x_smem) {
                // x and r rows per cluster that can be resident at once
                const int ncl = cg_max_clusters(c);
                if (!d_xg_) {
                    void* p = nullptr;
                    CK(cudaMalloc(&p, sizeof(double) * 2 * static_cast<size_t>(ncl) * pitch_));
                    gallocs_.push_back(p);
                    d_xg_ = static_cast<double*>(p);
                }
            }
            c.xg = d_xg_;
            if (c.glob) {
                // group mode: per group the exchange rows / partials, and one
                // sequence flag per CTA (cg_kernels.cuh)
                const size_t ng = static_cast<size_t>(cg_max_clusters(c));
                if (!d_gex_) {
                    const size_t per = cg_glob_doubles_per_group(c);
                    void* p = nullptr;
                    CK(cudaMalloc(&p, sizeof(double) * per * ng + sizeof(unsigned long long) * ng * c.cs));
                    CK(cudaMemset(p, 0, sizeof(double) * per * ng + sizeof(unsigned long long) * ng * c.cs));
                    gallocs_.push_back(p);
                    d_gex_ = static_cast<double*>(p);
                    d_gflag_ = reinterpret_cast<unsigned long long*>(d_gex_ + per * ng);
                }
                c.gex = d_gex_;
                c.gflag = d_gflag_;
            }
        } else {
            ScalarCoefDev& c = Lv.sco;
            if (kind_ == ATM_PHI_DAHLQUIST) {
                // dahlquist.hpp:36-42
                const double hh = dt / S;
                const double m = 1.0 / (1.0 - prob_.lambda * hh);
                double out = m;
                for (int ss = 1; ss < S; ++ss) out *= m;
                c.mult = out;
            } else {
                c.mult = prob_.mult[l];
            }
            c.ff = (folded_ && l == 0 && d_ff_) ? d_ff_ : nullptr;
        }
    }
}

// ---------------------------------------------------------------------------
// launch helpers

// output staging: double-buffered unless a single buffer buys occupancy
static int choose_n_out(SweepArgs a) {
    if (const char* e = std::getenv("ATM_NOUT")) return std::atoi(e) == 1 ? 1 : 2;
    a.n_out = 2;
    const int o2 = heat_sweep_occupancy(a);
    a.n_out = 1;
    const int o1 = heat_sweep_occupancy(a);
    return o1 > o2 ? 1 : 2;
}

int Engine::grid_for(int jobs, int occ) {
    if (jobs <= 0) return 0;
    return std::max(1, std::min(jobs, sms_ * std::max(1, occ)));
}

void Engine::check_launch(int err, const char* what) {
    ++launches_;
    if (err != 0)
        throw Error(ATM_RUNTIME_FAULT, std::string("kernel launch failed (") + what + "): " +
                                           cudaGetErrorString(static_cast<cudaError_t>(err)));
}

void Engine::phase_begin(const char* name) {
    if (!trace_) return;
    cudaEvent_t a, b;
    if (ev_pool_.size() >= 2) {
        a = ev_pool_.back(); ev_pool_.pop_back();
        b = ev_pool_.back(); ev_pool_.pop_back();
    } else {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    CK(cudaEventRecord(a, st_));
    Pending pe;
    pe.first = name;
    pe.second = {a, b};
    pending_.push_back(pe);
}

void Engine::phase_end() {
    if (!trace_ || pending_.empty()) return;
    // close the innermost open phase
    for (auto it = pending_.rbegin(); it != pending_.rend(); ++it) {
        if (!it->closed) {
            CK(cudaEventRecord(it->second.second, st_));
            it->closed = true;
            break;
        }
    }
}

// sweep jobs [j0, j1) on one shard/level
void Engine::sweep_jobs(Shard& s, int level, int kind, int j0, int j1, int tail, int m_override,
                        double* sq, int sq_base, int store) {
    if (j1 <= j0) return;
    LevelDev& Lv = s.lv[level];
    const int m = m_override > 0 ? m_override : H_.m[level];
    const bool add_g = Lv.g_full;
    LevelDev* out_lv =
        ((tail == TAIL_STORE || tail == TAIL_BOTH) && m_override <= 0) ? &s.lv[level + 1] : nullptr;
    if (heat_) {
        SweepArgs a{};
        a.co = Lv.hco;
        a.kind = kind;
        a.m = m;
        a.np = H_.np[level];
        a.j0 = j0;
        a.j1 = j1;
        a.u_base = Lv.u.base;
        a.u_div = Lv.u.div;
        a.g_base = add_g ? Lv.g.base : 0;
        a.add_g = add_g;
        a.forced = phi_forced_;
        a.store = store;
        a.tail = tail;
        a.out_base = out_lv ? out_lv->r.base : 0;
        a.sq = sq;
        a.sq_base = sq_base;
        a.sq_div = sq == d_sq_c_ ? H_.m[level] : 1;  // per-C-point stopping squares
        const CUtensorMap& tg = add_g ? Lv.g.tm : Lv.u.tm;
        const CUtensorMap& to = out_lv ? out_lv->r.tm : Lv.u.tm;
        a.n_out = choose_n_out(a);
        // streaming rows: an array several times the L2 cannot be re-read from it,
        // so its row stores are marked evict_first (config-5 correction sweep
        // 0.95 -> 1.00 of the measured HBM copy peak); smaller levels keep the
        // default policy
        a.st_hint = sizeof(double) * pitch_ * static_cast<size_t>(Lv.u.rows) > 2 * l2_bytes_ ? 1 : 0;
        if (const char* e = std::getenv("ATM_ST_HINT")) a.st_hint = std::atoi(e);
        int grid = grid_for(j1 - j0, heat_sweep_occupancy(a));
        if (const char* e = std::getenv("ATM_GRID_SWEEP")) grid = std::min(grid, std::atoi(e));
        if (std::getenv("ATM_DEBUG_OCC"))
            std::fprintf(stderr, "sweep level %d L %d nt %d n_out %d smem %zu occ %d grid %d\n", level,
                         a.co.L, a.co.nt, a.n_out, heat_sweep_smem(a), heat_sweep_occupancy(a), grid);
        const CUtensorMap& tow = out_lv ? out_lv->r.tmw : Lv.u.tmw;
        check_launch(launch_heat_sweep(a, Lv.u.tm, tg, to, Lv.u.tmw, tow, grid, st_), "heat_sweep");
    } else if (h2d_) {
        CgSweepArgs a{};
        a.co = Lv.gco;
        a.kind = kind;
        a.m = m;
        a.np = H_.np[level];
        a.j0 = j0;
        a.j1 = j1;
        a.u = Lv.u.p;
        a.u_base = Lv.u.base;
        a.u_div = Lv.u.div;
        a.g = add_g ? Lv.g.p : nullptr;
        a.g_base = add_g ? Lv.g.base : 0;
        a.add_g = add_g;
        a.forced = phi_forced_;
        a.store = store;
        a.tail = tail;
        a.out = out_lv ? out_lv->r.p : nullptr;
        a.out_base = out_lv ? out_lv->r.base : 0;
        a.sq = sq;
        a.sq_base = sq_base;
        a.sq_div = sq == d_sq_c_ ? H_.m[level] : 1;  // per-C-point stopping squares
        check_launch(launch_cg_sweep(a, st_), "cg_sweep");
    } else {
        ScalarSweepArgs a{};
        a.co = Lv.sco;
        a.kind = kind;
        a.m = m;
        a.np = H_.np[level];
        a.j0 = j0;
        a.j1 = j1;
        a.u = Lv.u.p;
        a.u_base = Lv.u.base;
        a.u_div = Lv.u.div;
        a.g = add_g ? Lv.g.p : nullptr;
        a.g_base = add_g ? Lv.g.base : 0;
        a.add_g = add_g;
        a.store = store;
        a.tail = tail;
        a.out = out_lv ? out_lv->r.p : nullptr;
        a.out_base = out_lv ? out_lv->r.base : 0;
        a.sq = sq;
        a.sq_base = sq_base;
        a.sq_div = sq == d_sq_c_ ? H_.m[level] : 1;  // per-C-point stopping squares
        check_launch(launch_scalar_sweep(a, st_), "scalar_sweep");
    }
}

void Engine::window_launch(Shard& s, int level, int kind, int pre_lo, int pre_e0, int pre_e1,
                           int p0, int p1, const DArr& x1, const DArr& x2, const DArr& x3,
                           const DArr& out, int out_stride, int forced, int seed_zero, int idx0,
                           int seed_off) {
    const bool has_pre = (kind <= WK_FORWARD) && pre_e1 >= pre_e0;
    const int jobs = (has_pre ? 1 : 0) + std::max(0, p1 - p0 + 1);
    if (jobs <= 0) return;
    LevelDev& Lv = s.lv[level];
    if (heat_) {
        WindowArgs a{};
        a.co = Lv.hco;
        a.kind = kind;
        a.k = H_.k;
        a.pre_lo = pre_lo;
        a.pre_e0 = pre_e0;
        a.pre_e1 = pre_e1;
        a.p0 = p0;
        a.p1 = p1;
        a.x1_base = x1.base;
        a.x2_base = x2.base;
        a.x3_base = x3.base;
        a.out_base = out.base;
        a.out_stride = out_stride;
        a.forced = forced && Lv.hco.theta != nullptr;  // heat1d: manufactured forcing only
        a.seed_zero = seed_zero;
        a.idx0 = idx0;
        a.seed_off = seed_off;
        // a long prefix chain alone in the launch (classical coarse grid,
        // k >= N_T + 1): its emits are sequential, so the next C row is
        // fetched two emits ahead (two more staging rows; the occupancy it
        // costs does not matter to a single chain)
        a.two_s = kind == WK_LINEAR && has_pre && pre_e1 - pre_e0 >= 64 && p1 < p0 &&
                  Lv.hco.L != 32 && !std::getenv("ATM_WIN_ONE_S");
        const CUtensorMap& t1 = x1.has_tm ? x1.tm : out.tm;
        const CUtensorMap& t2 = x2.has_tm ? x2.tm : t1;
        const CUtensorMap& t3 = x3.has_tm ? x3.tm : t1;
        int grid = grid_for(jobs, heat_window_occupancy(a));
        if (std::getenv("ATM_DEBUG_OCC"))
            std::fprintf(stderr, "window kind %d level %d L %d nt %d smem %zu occ %d grid %d\n", kind,
                         level, a.co.L, a.co.nt, heat_window_smem(a), heat_window_occupancy(a), grid);
        if (const char* e = std::getenv("ATM_GRID_WINDOW")) grid = std::min(grid, std::atoi(e));
        check_launch(launch_heat_window(a, t1, t2, t3, out.tm, grid, st_), "heat_window");
    } else if (h2d_) {
        CgWindowArgs a{};
        a.co = Lv.gco;
        a.kind = kind;
        a.k = H_.k;
        a.pre_lo = pre_lo;
        a.pre_e0 = pre_e0;
        a.pre_e1 = pre_e1;
        a.p0 = p0;
        a.p1 = p1;
        a.x1 = x1.p;
        a.x1_base = x1.base;
        a.x2 = x2.p;
        a.x2_base = x2.base;
        a.x3 = x3.p;
        a.x3_base = x3.base;
        a.out = out.p;
        a.out_base = out.base;
        a.out_stride = out_stride;
        a.forced = forced && d_src_ != nullptr;
        a.seed_zero = seed_zero;
        a.idx0 = idx0;
        a.seed_off = seed_off;
        check_launch(launch_cg_window(a, st_), "cg_window");
    } else {
        ScalarWindowArgs a{};
        a.co = Lv.sco;
        if (forced == 0 && kind == WK_APPLY) a.co.ff = Lv.sco.ff;
        a.kind = kind;
        a.k = H_.k;
        a.pre_lo = pre_lo;
        a.pre_e0 = pre_e0;
        a.pre_e1 = pre_e1;
        a.p0 = p0;
        a.p1 = p1;
        a.x1 = x1.p;
        a.x1_base = x1.base;
        a.x2 = x2.p;
        a.x2_base = x2.base;
        a.x3 = x3.p;
        a.x3_base = x3.base;
        a.out = out.p;
        a.out_base = out.base;
        a.out_stride = out_stride;
        a.seed_zero = seed_zero;
        a.idx0 = idx0;
        a.seed_off = seed_off;
        check_launch(launch_scalar_window(a, st_), "scalar_window");
    }
}

// ---------------------------------------------------------------------------
// exchanges (Execution hooks, solver.hpp:40-60)

void Engine::halo(int level, DArr LevelDev::*arr) {
    // sync_left_edge (parallel.cpp:236-249): u[lo-1] <- left neighbour's u[hi]
    if (G_ == 1) return;
    const size_t bytes = sizeof(double) * pitch_;
    if (world_ == 1) {
        for (Shard& s : sh_) {
            LevelDev& Lv = s.lv[level];
            if (Lv.hi < Lv.lo || Lv.lo == 0 || Lv.left < 0) continue;
            const DArr& src = sh_[Lv.left].lv[level].*arr;
            const DArr& dst = Lv.*arr;
            const int i = Lv.lo - 1;
            CK(cudaMemcpyAsync(dst.p + dst.off(i, pitch_),
                               src.p + src.off(i, pitch_), bytes,
                               cudaMemcpyDeviceToDevice, st_));
        }
        return;
    }
    Shard& s = sh_[0];
    LevelDev& Lv = s.lv[level];
    if (Lv.hi < Lv.lo) return;
    const DArr& a = Lv.*arr;
    ncclComm_t c = comm();
    nccl_->check(nccl_->GroupStart(), "group");
    if (Lv.right >= 0)
        nccl_->check(nccl_->Send(a.p + a.off(Lv.hi, pitch_), pitch_,
                                 ncclFloat64, Lv.right, c, st_), "send halo");
    if (Lv.lo > 0 && Lv.left >= 0)
        nccl_->check(nccl_->Recv(a.p + a.off(Lv.lo - 1, pitch_), pitch_,
                                 ncclFloat64, Lv.left, c, st_), "recv halo");
    nccl_->check(nccl_->GroupEnd(), "group");
}

// Window payloads (exchange_local_windows, parallel.cpp:134-194): each shard
// receives exactly the coarsest indices [max(0, lo-k+1), lo-1] it lacks.
void Engine::window_exchange(int level, DArr LevelDev::*arr) {
    if (G_ == 1) return;
    const int k = H_.k;
    const size_t rowb = sizeof(double) * pitch_;
    if (world_ == 1) {
        for (Shard& s : sh_) {
            LevelDev& Lv = s.lv[level];
            if (Lv.hi < Lv.lo) continue;
            const int need_lo = std::max(0, Lv.lo - k + 1);
            for (int j = need_lo; j < Lv.lo; ++j) {
                const int o = lay_.owner_of_coarse(j);
                const DArr& src = sh_[o].lv[level].*arr;
                const DArr& dst = Lv.*arr;
                CK(cudaMemcpyAsync(dst.p + dst.off(j, pitch_),
                                   src.p + src.off(j, pitch_), rowb,
                                   cudaMemcpyDeviceToDevice, st_));
            }
        }
        return;
    }
    Shard& s = sh_[0];
    LevelDev& Lv = s.lv[level];
    const DArr& a = Lv.*arr;
    ncclComm_t c = comm();
    nccl_->check(nccl_->GroupStart(), "group");
    for (int q = 0; q < G_; ++q) {
        if (q == rank_) continue;
        const Ranges& rq = ranges_all_[q];
        // what q needs from me
        const int q_lo = rq.lo[level];
        const int q_need_lo = std::max(0, q_lo - k + 1), q_need_hi = q_lo - 1;
        const int a0 = std::max(q_need_lo, Lv.lo), a1 = std::min(q_need_hi, Lv.hi);
        if (a1 >= a0 && Lv.hi >= Lv.lo)
            nccl_->check(nccl_->Send(a.p + a.off(a0, pitch_),
                                     static_cast<size_t>(a1 - a0 + 1) * pitch_, ncclFloat64, q, c,
                                     st_), "send window");
        // what I need from q
        const int my_need_lo = std::max(0, Lv.lo - k + 1), my_need_hi = Lv.lo - 1;
        const int b0 = std::max(my_need_lo, rq.lo[level]), b1 = std::min(my_need_hi, rq.hi[level]);
        if (b1 >= b0 && Lv.hi >= Lv.lo)
            nccl_->check(nccl_->Recv(a.p + a.off(b0, pitch_),
                                     static_cast<size_t>(b1 - b0 + 1) * pitch_, ncclFloat64, q, c,
                                     st_), "recv window");
    }
    nccl_->check(nccl_->GroupEnd(), "group");
    (void)rowb;
}

ncclComm_t Engine::comm() const {
    if (!comm_) throw Error(ATM_RUNTIME_FAULT, "rank " + std::to_string(rank_) + ": the NCCL communicator "
                                               "was aborted after an earlier fault");
    return static_cast<ncclComm_t>(comm_);
}

void Engine::sync_stream(const char* what) {
    if (world_ == 1 || !comm_) {
        CK(cudaStreamSynchronize(st_));
        return;
    }
    // polled wait: a peer that died or stalls leaves an NCCL kernel spinning on
    // this stream; fail like the reference's receive timeout (transport.cpp:
    // 29-48 -> RuntimeFault) instead of hanging, after aborting the communicator
    // so the stream drains (parallel.cpp:349-351: abort wakes the other ranks)
    // The common case is a wait of tens of microseconds on the critical path
    // of every iteration (the norm read-back): spin on the stream for the
    // first 2 ms without sleeping, and look at the clock, NCCL's error state
    // and the deadline only every 64 polls; a long wait then backs off to
    // 20 us sleeps.
    const auto t_start = std::chrono::steady_clock::now();
    const auto deadline = t_start + std::chrono::milliseconds(timeout_ms_);
    const auto spin_until = t_start + std::chrono::milliseconds(2);
    bool spinning = true;
    for (unsigned poll = 1;; ++poll) {
        const cudaError_t e = cudaStreamQuery(st_);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) ck(e, what);
        if (spinning && (poll & 63u)) continue;
        const auto now = std::chrono::steady_clock::now();
        if (spinning && now < spin_until) continue;
        spinning = false;
        std::string why;
        if (nccl_->GetAsyncError) {
            ncclResult_t ar = ncclSuccess;
            nccl_->GetAsyncError(static_cast<ncclComm_t>(comm_), &ar);
            if (ar != ncclSuccess && ar != ncclInProgress)
                why = std::string("NCCL asynchronous error: ") + nccl_->ErrStr(ar);
        }
        if (why.empty() && now > deadline)
            why = "timed out after " + std::to_string(timeout_ms_) + " ms";
        if (!why.empty()) {
            if (nccl_->Abort) nccl_->Abort(static_cast<ncclComm_t>(comm_));
            comm_ = nullptr;  // aborted: never used again (the destructor skips it)
            throw Error(ATM_RUNTIME_FAULT, "rank " + std::to_string(rank_) + ": " + why +
                                               " waiting for " + what + " (a peer rank failed or stalled)");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

double Engine::reduce_norm(double* sq, int count) {
    // world > 1: each rank's per-point array holds only its own points (the
    // rest stay 0 and are never written), so the element-wise sum is exact.
    // The sum goes to a separate buffer: reducing in place would leave the
    // other ranks' values in this rank's array for the next iteration.
    if (world_ > 1) {
        nccl_->check(nccl_->AllReduce(sq, d_sq_all_, count, ncclFloat64, ncclSum,
                                      comm(), st_), "allreduce squares");
        sq = d_sq_all_;
    }
    check_launch(launch_norm_from_squares(sq, count, d_norm_, st_), "norm");
    double out = 0.0;
    CK(cudaMemcpyAsync(&out, d_norm_, sizeof(double), cudaMemcpyDeviceToHost, st_));
    sync_stream("the residual norm");
    return out;
}

// ---------------------------------------------------------------------------
// setup (solver.cpp:81-150)

void Engine::fill_initial_guess() {
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[0];
        if (Lv.hi < Lv.lo) continue;
        const int dv = Lv.u.div;
        // C-point storage: the held points i0, i0 + dv, ... < i1
        const int i0 = (std::max(1, Lv.lo) + dv - 1) / dv * dv, i1 = Lv.hi + 1;
        const int nrows = i1 > i0 ? (i1 - i0 + dv - 1) / dv : 0;
        if (Lv.lo == 0)
            check_launch(launch_fill_rows(Lv.u.p, Lv.u.base, pitch_, n_, 0, 1, d_ic_, st_), "fill ic");
        switch (sol_.initial_guess) {
            case ATM_GUESS_CONSTANT: {
                double* v = d_ic_;
                if (!cval_.empty()) {
                    void* p = nullptr;
                    CK(cudaMalloc(&p, sizeof(double) * n_));
                    Lv.allocs.push_back(p);
                    CK(cudaMemcpy(p, cval_.data(), sizeof(double) * n_, cudaMemcpyHostToDevice));
                    v = static_cast<double*>(p);
                }
                if (nrows > 0)
                    check_launch(launch_fill_rows(Lv.u.p + Lv.u.off(i0, pitch_), 0, pitch_, n_, 0, nrows,
                                                  v, st_), "fill const");
                break;
            }
            case ATM_GUESS_RANDOM:
                check_launch(launch_fill_random(Lv.u.p, Lv.u.base, pitch_, n_, i0, i1, sol_.seed, st_, dv),
                             "fill random");
                break;
            case ATM_GUESS_PROVIDED:
                if (nrows > 0 && dv == 1 && H_.L >= 2 && H_.m[0] > 1 && rt_.defer_guess) {
                    // Only the C rows go now. Every cycle opens with an
                    // F-relaxation from the C points (kernels.cpp:7-17) and
                    // its correction F-sweep rewrites every F row before
                    // anything reads one, so the guess's F values are dead
                    // under cycling; an access that could see them first
                    // (residual_norm, level-0 reads/writes, kernel-level
                    // entry points, nested init) copies them (flush_guess).
                    const int m = H_.m[0];
                    const int c0 = (i0 + m - 1) / m * m;
                    const int nc = c0 < i1 ? (i1 - 1 - c0) / m + 1 : 0;
                    if (nc > 0)
                        CK(cudaMemcpy2DAsync(Lv.u.p + Lv.u.off(c0, pitch_), sizeof(double) * pitch_ * m,
                                             prov_ptr_ + static_cast<size_t>(c0) * n_,
                                             sizeof(double) * n_ * m, sizeof(double) * n_, nc,
                                             cudaMemcpyHostToDevice, st_));
                    h2d_bytes_ += sizeof(double) * n_ * static_cast<size_t>(nc);
                    guess_pending_ = true;
                } else if (nrows > 0) {
                    CK(cudaMemcpy2DAsync(Lv.u.p + Lv.u.off(i0, pitch_),
                                         sizeof(double) * pitch_, prov_ptr_ + static_cast<size_t>(i0) * n_,
                                         sizeof(double) * n_ * dv, sizeof(double) * n_, nrows,
                                         cudaMemcpyHostToDevice, st_));
                    h2d_bytes_ += sizeof(double) * n_ * static_cast<size_t>(nrows);
                }
                break;
        }
    }
}

// the deferred F rows of a provided guess (full level-0 storage only)
void Engine::flush_guess() {
    if (!guess_pending_) return;
    guess_pending_ = false;
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[0];
        if (Lv.hi < Lv.lo) continue;
        const int i0 = std::max(1, Lv.lo), i1 = Lv.hi + 1;
        if (i1 <= i0) continue;
        CK(cudaMemcpy2DAsync(Lv.u.p + Lv.u.off(i0, pitch_), sizeof(double) * pitch_,
                             prov_ptr_ + static_cast<size_t>(i0) * n_, sizeof(double) * n_,
                             sizeof(double) * n_, i1 - i0, cudaMemcpyHostToDevice, st_));
        h2d_bytes_ += sizeof(double) * n_ * static_cast<size_t>(i1 - i0);
    }
    sync_stream(__func__);
}

void Engine::fill_level_rhs(int level) {
    // g_0 = IC; g_i = 0 (folded) or forcing(level, i)  (solver.cpp:136-150)
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[level];
        if (Lv.hi < Lv.lo) continue;
        if (Lv.g.p && Lv.g.base == 0 && Lv.lo <= 1)
            check_launch(launch_fill_rows(Lv.g.p, Lv.g.base, pitch_, n_, 0, 1, d_ic_, st_), "g0");
        if (!Lv.g_full) continue;
        const int i0 = std::max(1, Lv.lo), i1 = Lv.hi;
        if (folded_) {
            if (i1 >= i0)
                CK(cudaMemsetAsync(Lv.g.p + Lv.g.off(i0, pitch_), 0,
                                   sizeof(double) * pitch_ * (i1 - i0 + 1), st_));
        } else if (heat_) {
            // forcing(level, i) = propagate(zero, with forcing) (heat1d.cpp:97-100)
            window_launch(s, level, WK_APPLY, 0, 0, -1, i0, i1, Lv.g, Lv.g, Lv.g, Lv.g, 1, 1, 1, 0, 0);
        } else if (h2d_) {
            // heat2d forcing is the same for every i (time-independent source):
            // one CG solve, then copies
            if (i1 >= i0) {
                window_launch(s, level, WK_APPLY, 0, 0, -1, i0, i0, Lv.g, Lv.g, Lv.g, Lv.g, 1, 1, 1, 0, 0);
                if (i1 > i0)
                    check_launch(launch_fill_rows(Lv.g.p, Lv.g.base, pitch_, n_, i0 + 1, i1 + 1,
                                                  Lv.g.p + Lv.g.off(i0, pitch_),
                                                  st_), "g rows");
            }
        } else {
            // scalar fixture: forcing(0, i) = ff[i] (tests/support.hpp:43-49)
            std::vector<double> rows(static_cast<size_t>(i1 - i0 + 1), 0.0);
            for (int i = i0; i <= i1; ++i)
                rows[i - i0] = (level == 0 && i < static_cast<int>(ff_.size())) ? ff_[i] : 0.0;
            if (i1 >= i0)
                CK(cudaMemcpyAsync(Lv.g.p + (i0 - Lv.g.base), rows.data(), sizeof(double) * rows.size(),
                                   cudaMemcpyHostToDevice, st_));
            sync_stream(__func__);
        }
    }
}

void Engine::setup() {
    if (setup_done_) return;
    phase_begin("fill");
    fill_initial_guess();
    fill_level_rhs(0);
    if (sol_.norm == ATM_NORM_FUNCTIONAL) {
        // prev_functional_ (solver.cpp:101-106): f of every own C point of the guess
        for (Shard& s : sh_) {
            LevelDev& Lv = s.lv[0];
            if (Lv.c_count > 0)
                check_launch(launch_functional(Lv.u.p, Lv.u.base / Lv.u.div, H_.m[0] / Lv.u.div, pitch_,
                                               n_, d_fw_, d_prevf_, Lv.c_first, Lv.c_first + Lv.c_count,
                                               nullptr, 1, st_),
                             "functional init");
        }
    }
    phase_end();
    sync_stream(__func__);
    setup_done_ = true;
}

// ---------------------------------------------------------------------------
// cycle pieces

void Engine::point0_residual(Shard& s, int level, double* r_out, double* sq_out) {
    // r_0 = g_0 - u_0 (kernels.cpp:35-37)
    LevelDev& Lv = s.lv[level];
    if (Lv.lo != 0 || Lv.hi < 0) return;
    const double* g0 = Lv.g.p;  // row 0 in both layouts (base == 0)
    check_launch(launch_row_diff(r_out, g0, Lv.u.p, n_, sq_out, st_), "r0");
}

// F-relaxation over own intervals (kernels.cpp:7-17) with optional tail
void Engine::f_sweep(int level, int tail, int store) {
    if (level == 0 && cpts_) {
        // C-point storage: level-0 F rows are never stored, so a sweep
        // without a tail has no observable result
        if (tail == TAIL_NONE) return;
        store = STORE_NONE;
    }
    // (the exchange of the previous cycle's correction sweep still stands when
    // no C point has been written since: halo0_valid_)
    if (!(level == 0 && halo0_valid_)) halo(level, &LevelDev::u);
    const char* tag = level != 0 ? nullptr
                      : (tail == TAIL_SQ || tail == TAIL_BOTH) ? "sweep_correct"
                      : tail == TAIL_STORE                     ? "sweep_relax"
                                                               : "sweep_f";
    if (tag) phase_begin(tag);
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[level];
        if (Lv.iv_count == 0) continue;
        sweep_jobs(s, level, SW_F, Lv.iv_first, Lv.iv_first + Lv.iv_count, tail, 0,
                   (tail == TAIL_SQ || tail == TAIL_BOTH) ? d_sq_c_ : nullptr, 0, store);
    }
    if (tag) phase_end();
}

// relax_level (solver.cpp:160-172).  With F-relaxation the restriction
// residuals are produced by the sweep's tail.
void Engine::relax_level(int level, bool restrict_tail, bool f_dead) {
    // F rows a later pass still reads: none with F-relaxation (the residual
    // comes from the sweep's tail), the last F row of every interval otherwise
    const int fst = !f_dead ? STORE_ALL : sol_.relaxation == ATM_RELAX_F ? STORE_NONE : STORE_CF;
    if (sol_.relaxation == ATM_RELAX_F) {
        f_sweep(level, restrict_tail ? TAIL_STORE : TAIL_NONE, fst);
        return;
    }
    if (sol_.nu == 1) {
        // fused F-C-F: job J chains from the old C_{J-1} through the
        // C-relaxation of C_J into interval J (kernels.cpp:7-28)
        halo(level, &LevelDev::u);
        for (Shard& s : sh_) {
            LevelDev& Lv = s.lv[level];
            if (Lv.c_count == 0) continue;
            int j1 = Lv.c_first + Lv.c_count;
            sweep_jobs(s, level, SW_FCF, Lv.c_first, j1, TAIL_NONE, 0, nullptr, 0, fst);
        }
        if (G_ > 1) {
            // the first interval of a shard waits for its left neighbour's new C
            halo(level, &LevelDev::u);
            for (Shard& s : sh_) {
                LevelDev& Lv = s.lv[level];
                if (Lv.iv_count == 0 || Lv.iv_first >= Lv.c_first) continue;
                sweep_jobs(s, level, SW_F, Lv.iv_first, Lv.iv_first + 1, TAIL_NONE, 0, nullptr, 0,
                           fst);
            }
        }
        return;
    }
    f_sweep(level, TAIL_NONE, fst);
    for (int it = 0; it < sol_.nu; ++it) {
        for (Shard& s : sh_) {
            LevelDev& Lv = s.lv[level];
            const int j0 = std::max(1, Lv.c_first), j1 = Lv.c_first + Lv.c_count;
            sweep_jobs(s, level, SW_CRELAX, j0, j1, TAIL_NONE, 0, nullptr, 0);
        }
        f_sweep(level, TAIL_NONE, fst);
    }
}

// residual at own C-points of `level` into level+1 r (solver.cpp:307-314)
void Engine::resid_c(int level) {
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[level];
        if (Lv.c_count == 0) continue;
        const int j0 = std::max(1, Lv.c_first), j1 = Lv.c_first + Lv.c_count;
        sweep_jobs(s, level, SW_RESID, j0, j1, TAIL_STORE, 0, nullptr, 0);
    }
}

void Engine::restrict_to(int level) {
    // solver.cpp:194-222
    const int lc = H_.coarsest();
    const int m = H_.m[level];
    const bool relaxed = (level + 1) != lc;
    if (sol_.relaxation != ATM_RELAX_F) resid_c(level);
    if (sol_.relaxation != ATM_RELAX_F && G_ > 1) halo(level, &LevelDev::u);
    for (Shard& s : sh_) {
        LevelDev& F = s.lv[level];
        LevelDev& C = s.lv[level + 1];
        if (F.c_count == 0) continue;
        const int j0 = F.c_first, cnt = F.c_count;
        // injection: coarse u = coarse v = fine u at C-points (kernels.cpp:45-51)
        const size_t rowb = sizeof(double) * pitch_;
        const double* src = F.u.p + F.u.off(j0 * m, pitch_);
        for (DArr* dst : {&C.u, &C.v})
            CK(cudaMemcpy2DAsync(dst->p + dst->off(j0, pitch_), rowb, src,
                                 rowb * (m / F.u.div), rowb, cnt, cudaMemcpyDeviceToDevice, st_));
        if (j0 > 0 && C.v.valid(j0 - 1) && F.u.valid((j0 - 1) * m))
            CK(cudaMemcpyAsync(C.v.p + C.v.off(j0 - 1, pitch_),
                               F.u.p + F.u.off((j0 - 1) * m, pitch_), rowb,
                               cudaMemcpyDeviceToDevice, st_));
        if (j0 == 0) point0_residual(s, level, C.r.p, nullptr);
        if (relaxed) {
            // g_j = (v_j - Psi_j(v_{j-1})) + r_j, j >= 1; g_0 = v_0 + r_0
            const int p0 = std::max(1, j0), p1 = j0 + cnt - 1;
            window_launch(s, level + 1, WK_FAS_RHS, 0, 0, -1, p0, p1, C.v, C.v, C.r, C.g, 1,
                          phi_forced_, 0, 0, 0);
            if (j0 == 0)
                check_launch(launch_row_sum(C.g.p, C.v.p, C.r.p, n_, st_), "g0 fas");
        }
    }
}

void Engine::windows(int kind) {
    if (std::getenv("ATM_SYNC_PHASES")) CK(cudaDeviceSynchronize());
    // coarsest_linear / coarsest_fas / nested forward (solver.cpp:224-279, :347-356)
    const int lc = H_.coarsest();
    const int k = H_.k;
    for (Shard& s : sh_) {
        LevelDev& C = s.lv[lc];
        if (C.hi < C.lo) continue;
        const int plo = C.lo, phi = C.hi;
        // windows with lo = 0 (p <= k-1) share one prefix chain
        const int pre_e0 = plo, pre_e1 = std::min(k - 1, phi);
        const int p0 = std::max(plo, k), p1 = phi;
        const int forced = phi_forced_;
        if (kind == WK_LINEAR) {
            // the corrections land on level-0 C rows: row p * m - base, or
            // p - base / m with C-point storage
            DArr out = s.lv[0].u;
            out.base /= out.div;
            window_launch(s, lc, WK_LINEAR, 0, pre_e0, pre_e1, p0, p1, C.r, C.r, C.r, out,
                          H_.m[0] / s.lv[0].u.div, forced, 0, 0, 0);
        } else if (kind == WK_FAS) {
            // Psi(v_{j-1}) once per coarse point, shared by every window
            const int a0 = std::max(1, C.base + 1);
            window_launch(s, lc, WK_APPLY, 0, 0, -1, a0, phi, C.v, C.v, C.v, C.w, 1, forced, 0, 0, -1);
            window_launch(s, lc, WK_FAS, 0, pre_e0, pre_e1, p0, p1, C.r, C.v, C.w, C.u, 1, forced,
                          0, 0, 0);
        } else {
            window_launch(s, lc, WK_FORWARD, 0, pre_e0, pre_e1, p0, p1, C.x, C.x, C.x, C.u, 1,
                          forced, 0, 0, 0);
        }
    }
}

void Engine::coarsest_linear() {
    phase_begin("exchange");
    window_exchange(1, &LevelDev::r);
    phase_end();
    phase_begin("coarse");
    windows(WK_LINEAR);
    phase_end();
}

void Engine::coarsest_fas() {
    const int lc = H_.coarsest();
    phase_begin("exchange");
    window_exchange(lc, &LevelDev::v);
    window_exchange(lc, &LevelDev::r);
    phase_end();
    phase_begin("coarse");
    windows(WK_FAS);
    phase_end();
}

void Engine::correct_from(int level) {
    // solver.cpp:281-292
    const int m = H_.m[level];
    for (Shard& s : sh_) {
        LevelDev& F = s.lv[level];
        LevelDev& C = s.lv[level + 1];
        if (F.c_count == 0) continue;
        check_launch(launch_c_correct(F.u.p, F.u.base / F.u.div, m / F.u.div, C.u.p, C.v.p, C.u.base,
                                      pitch_, n_, F.c_first, F.c_first + F.c_count, st_), "c_correct");
    }
    f_sweep(level, level != 0 ? TAIL_NONE : reuse_possible() ? TAIL_BOTH : TAIL_SQ);
    if (level == 0)
        for (Shard& s : sh_) point0_residual(s, 0, d_row_, d_sq_c_);
}

void Engine::v_cycle(int level) {
    // solver.cpp:294-303
    if (level == H_.coarsest()) {
        coarsest_fas();
        return;
    }
    // relax reuse (level 0 only): the opening F-sweep would recompute what the
    // previous cycle's correction sweep left, and its residuals are stored
    phase_begin("relax");
    if (!(level == 0 && reuse_possible() && relax_valid_))
        relax_level(level, sol_.relaxation == ATM_RELAX_F, true);
    phase_end();
    phase_begin("restrict");
    restrict_to(level);
    phase_end();
    v_cycle(level + 1);
    phase_begin("correct");
    correct_from(level);
    phase_end();
}

// Relax reuse (opt-in, atm_runtime.reuse_relax): with F-relaxation, a
// cycle's opening level-0 F-sweep recomputes from the same C points exactly
// what the previous cycle's level-0 correction F-sweep computed, and its only
// consumed output is the restriction residual at the C points.  The
// correction sweep then also stores those residuals into level 1's r
// (TAIL_BOTH; nothing reads r between the restriction and the end of the
// cycle) and the next cycle skips its F-sweep -- bitwise the same cycle, in
// the two-level cycle and on level 0 of the FAS V-cycle alike (the coarser
// levels' states are re-injected every cycle, so only level 0 repeats).
bool Engine::reuse_possible() const {
    return rt_.reuse_relax && sol_.relaxation == ATM_RELAX_F && H_.L >= 2;
}

void Engine::two_level_cycle() {
    // solver.cpp:305-320
    const bool reuse = reuse_possible();
    phase_begin("relax");
    if (!(reuse && relax_valid_)) relax_level(0, sol_.relaxation == ATM_RELAX_F, true);
    phase_end();
    phase_begin("restrict");
    if (sol_.relaxation != ATM_RELAX_F) resid_c(0);
    for (Shard& s : sh_) point0_residual(s, 0, s.lv[1].r.p, nullptr);
    phase_end();
    halo0_valid_ = false;  // the windows write the C points
    coarsest_linear();
    phase_begin("correct");
    f_sweep(0, reuse ? TAIL_BOTH : TAIL_SQ);
    for (Shard& s : sh_) point0_residual(s, 0, d_row_, d_sq_c_);
    phase_end();
    relax_valid_ = reuse;
    // one process per shard (no graph replay of a fixed exchange sequence):
    // the correction sweep's halo serves the next cycle's relaxation sweep too
    halo0_valid_ = world_ > 1 && sol_.relaxation == ATM_RELAX_F && !std::getenv("ATM_HALO_EVERY_SWEEP");
}

// One cycle = a fixed launch sequence on one stream: captured once into a
// CUDA graph and replayed (small configs are launch-bound).
// Not with phase tracing (host-side event bookkeeping), multi-process NCCL,
// or the Newton / CG families (their failure flag is read back every cycle).
bool Engine::use_graphs() const {
    if (world_ > 1 || trace_ || ac_ || h2d_) return false;
    return !std::getenv("ATM_NO_GRAPH") && !std::getenv("ATM_SYNC_PHASES");
}

void Engine::cycle() {
    setup();
    launches_ = 0;
    // with relax reuse the first cycle (which still runs the opening F-sweep)
    // is not the steady-state launch sequence: capture from the second on
    const bool graphs = use_graphs() && (!reuse_possible() || relax_valid_);
    if (graphs && graph_exec_) {
        CK(cudaGraphLaunch(graph_exec_, st_));
        last_launches_ = graph_launches_;
        return;
    }
    if (graphs) CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    try {
        if (sol_.mode == ATM_TWO_LEVEL) {
            two_level_cycle();
        } else {
            v_cycle(0);
            relax_valid_ = reuse_possible();
        }
    } catch (...) {
        relax_valid_ = halo0_valid_ = false;
        if (graphs) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(st_, &g);
            if (g) cudaGraphDestroy(g);
        }
        // the cycle's correction F-sweep (which rewrites every level-0 F row)
        // may not have been enqueued: the deferred F rows of a provided guess
        // must land, so the state reads as it would after an eager copy
        if (guess_pending_) {
            try {
                flush_guess();
            } catch (...) {
            }
        }
        throw;
    }
    // every level-0 F row is rewritten by this cycle before anything reads it
    // (also when check_newton below throws: the kernels ran to completion)
    guess_pending_ = false;
    if (graphs) {
        cudaGraph_t g = nullptr;
        CK(cudaStreamEndCapture(st_, &g));
        const cudaError_t e = cudaGraphInstantiate(&graph_exec_, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        graph_launches_ = launches_;
        CK(cudaGraphLaunch(graph_exec_, st_));
    }
    last_launches_ = launches_;
    try {
        check_newton();
    } catch (...) {
        relax_valid_ = halo0_valid_ = false;  // a failed Phi leaves no residuals worth keeping
        throw;
    }
}

// NonlinearSolveError (gray_scott.cpp:165-169 analogue): a Newton solve hit
// newton_max somewhere in the last batch of Allen-Cahn Phi applications
void Engine::check_newton() {
    if (!ac_ && !h2d_) return;
    int f = 0;
    CK(cudaMemcpyAsync(&f, d_fail_, sizeof(int), cudaMemcpyDeviceToHost, st_));
    sync_stream(__func__);
    if (f) {
        CK(cudaMemsetAsync(d_fail_, 0, sizeof(int), st_));
        if (gs_)
            throw Error(ATM_NONLINEAR_FAIL, f == 2 ? "gray-scott: concentration left the bounding box"
                                                   : "gray-scott: Newton or the inner BiCGSTAB failed");
        if (h2d_)
            throw Error(ATM_NONLINEAR_FAIL, "heat2d: CG did not converge in " +
                                                std::to_string(prob_.cg_max) + " iterations");
        throw Error(ATM_NONLINEAR_FAIL, "allen-cahn: Newton did not converge in " +
                                            std::to_string(prob_.newton_max) + " iterations");
    }
}

void Engine::nested_init() {
    // solver.cpp:331-368
    setup();
    flush_guess();
    relax_valid_ = halo0_valid_ = false;
    const int lc = H_.coarsest();
    for (int l = 0; l < lc; ++l) {
        const int m = H_.m[l];
        for (Shard& s : sh_) {
            LevelDev& F = s.lv[l];
            LevelDev& C = s.lv[l + 1];
            if (F.c_count == 0) continue;
            const size_t rowb = sizeof(double) * pitch_;
            CK(cudaMemcpy2DAsync(C.u.p + C.u.off(F.c_first, pitch_), rowb,
                                 F.u.p + F.u.off(F.c_first * m, pitch_),
                                 rowb * (m / F.u.div), rowb, F.c_count, cudaMemcpyDeviceToDevice, st_));
        }
        fill_level_rhs(l + 1);
    }
    const int forced = phi_forced_;
    if (H_.k >= H_.np[lc]) {
        // chain_forward: sequential across shards (parallel.cpp:257-277)
        for (size_t si = 0; si < sh_.size(); ++si) {
            Shard& s = sh_[si];
            LevelDev& C = s.lv[lc];
            if (C.hi < C.lo) continue;
            if (world_ == 1 && C.lo > 0) {
                const DArr& src = sh_[C.left].lv[lc].u;
                CK(cudaMemcpyAsync(C.u.p + C.u.off(C.lo - 1, pitch_),
                                   src.p + src.off(C.lo - 1, pitch_),
                                   sizeof(double) * pitch_, cudaMemcpyDeviceToDevice, st_));
            } else if (world_ > 1 && C.lo > 0) {
                nccl_->check(nccl_->Recv(C.u.p + C.u.off(C.lo - 1, pitch_),
                                         pitch_, ncclFloat64, C.left, comm(), st_),
                             "chain recv");
            }
            const int from = std::max(0, C.lo - 1);
            window_launch(s, lc, WK_FORWARD, from, std::max(1, C.lo), C.hi, 1, 0, C.u, C.u, C.u,
                          C.u, 1, forced, 0, 0, 0);
            if (world_ > 1 && C.right >= 0)
                nccl_->check(nccl_->Send(C.u.p + C.u.off(C.hi, pitch_), pitch_,
                                         ncclFloat64, C.right, comm(), st_),
                             "chain send");
        }
    } else {
        for (Shard& s : sh_) {
            LevelDev& C = s.lv[lc];
            if (C.hi < C.lo) continue;
            CK(cudaMemcpyAsync(C.x.p + C.x.off(C.lo, pitch_),
                               C.u.p + C.u.off(C.lo, pitch_),
                               sizeof(double) * pitch_ * (C.hi - C.lo + 1), cudaMemcpyDeviceToDevice, st_));
        }
        window_exchange(lc, &LevelDev::x);
        windows(WK_FORWARD);
    }
    for (int l = lc - 1; l >= 0; --l) {
        const int m = H_.m[l];
        for (Shard& s : sh_) {
            LevelDev& F = s.lv[l];
            LevelDev& C = s.lv[l + 1];
            if (F.c_count == 0) continue;
            const size_t rowb = sizeof(double) * pitch_;
            CK(cudaMemcpy2DAsync(F.u.p + F.u.off(F.c_first * m, pitch_),
                                 rowb * (m / F.u.div), C.u.p + C.u.off(F.c_first, pitch_),
                                 rowb, rowb, F.c_count, cudaMemcpyDeviceToDevice, st_));
        }
        f_sweep(l, TAIL_NONE);
        if (l >= 1) v_cycle(l);
    }
    sync_stream(__func__);
    check_newton();
}

double Engine::residual_norm() {
    // full residual over all level-0 points (solver.cpp:370-378), m = 1 jobs
    setup();
    flush_guess();
    phase_begin("norm");
    halo(0, &LevelDev::u);
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[0];
        if (Lv.hi < Lv.lo) continue;
        if (cpts_) {
            // held F values are by definition the F-relaxation of their C
            // point (zero residual): only the C-point residuals remain
            if (Lv.iv_count > 0)
                sweep_jobs(s, 0, SW_F, Lv.iv_first, Lv.iv_first + Lv.iv_count, TAIL_SQ, 0, d_sq_full_, 0,
                           STORE_NONE);
        } else {
            sweep_jobs(s, 0, SW_RESID, std::max(1, Lv.lo), Lv.hi + 1, TAIL_SQ, 1, d_sq_full_, 0);
        }
        point0_residual(s, 0, d_row_, d_sq_full_);
    }
    const double v = reduce_norm(d_sq_full_, H_.np[0]);
    phase_end();
    return v;
}

double Engine::functional_change() {
    double mx = 0.0;
    for (size_t i = 0; i < sh_.size(); ++i) {
        LevelDev& Lv = sh_[i].lv[0];
        if (Lv.c_count == 0) continue;
        check_launch(launch_functional(Lv.u.p, Lv.u.base / Lv.u.div, H_.m[0] / Lv.u.div, pitch_, n_,
                                       d_fw_, d_prevf_, Lv.c_first, Lv.c_first + Lv.c_count,
                                       d_fmax_ + i, 0, st_), "functional");
    }
    if (world_ > 1)
        nccl_->check(nccl_->AllReduce(d_fmax_, d_fmax_, 1, ncclFloat64, ncclMax,
                                      comm(), st_), "allreduce max");
    std::vector<double> h(sh_.size(), 0.0);
    CK(cudaMemcpyAsync(h.data(), d_fmax_, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st_));
    sync_stream(__func__);
    for (double v : h) mx = std::max(mx, v);
    return mx;
}

double Engine::stopping_norm_after_cycle() {
    // stopping_norm (solver.cpp:380-396).  After a cycle every F-point
    // residual is bitwise zero (the last operation on each F-point is the
    // correction F-relaxation from its predecessor), so the C-point squares
    // written by the correction sweep's tail are the full per-point array.
    if (sol_.norm == ATM_NORM_FUNCTIONAL) return functional_change();
    phase_begin("norm");
    const double v = reduce_norm(d_sq_c_, H_.n_c(0));
    phase_end();
    return v;
}

double Engine::iterate_timed(int count, double* norms) {
    setup();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    sync_stream(__func__);
    CK(cudaEventRecord(a, st_));
    for (int i = 0; i < count; ++i) {
        cycle();
        const double v = stopping_norm_after_cycle();
        if (norms) norms[i] = v;
    }
    CK(cudaEventRecord(b, st_));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

void Engine::iterate(int count, double* norms) {
    setup();
    for (int i = 0; i < count; ++i) {
        cycle();
        const double v = stopping_norm_after_cycle();
        if (norms) norms[i] = v;
    }
}

void Engine::host_phase(const char* name, double seconds) {
    phase_sec_[name] += seconds;
    phase_cnt_[name] += 1;
}

int Engine::solve(atm_report* rep, double* norms, double* iter_secs) {
    // drive (solver.cpp:398-435)
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    setup();
    if (sol_.mode == ATM_NESTED_V) nested_init();
    const auto t_setup = clock::now();
    const double setup_s = std::chrono::duration<double>(t_setup - t0).count();
    host_phase("setup", setup_s);
    atm_report r{};
    r.setup_seconds = setup_s;
    r.stop_reason = 1;
    double dof_steps = 0.0;
    int status = ATM_NOT_CONVERGED;
    for (int it = 1; it <= sol_.max_iters; ++it) {
        const auto t_it = clock::now();
        cycle();
        const double v = stopping_norm_after_cycle();  // one device->host read: synchronised
        if (iter_secs) iter_secs[it - 1] = std::chrono::duration<double>(clock::now() - t_it).count();
        if (norms) norms[it - 1] = v;
        r.iterations = it;
        // relaxation Phi applications: every F-point twice per level visit
        // (once when the opening F-sweep is reused)
        const bool reused = reuse_possible() && it > 1;
        for (int l = 0; l + 1 < H_.L; ++l) {
            const double F = static_cast<double>(H_.np[l] - H_.n_c(l));
            double per = (reused && l == 0) ? F : 2.0 * F;
            if (sol_.relaxation == ATM_RELAX_FCF) per += sol_.nu * (F + H_.n_c(l) - 1);
            dof_steps += per * n_;
        }
        if (!std::isfinite(v)) {
            r.stop_reason = 2;
            r.total_seconds = std::chrono::duration<double>(clock::now() - t0).count();
            host_phase("iterations", std::chrono::duration<double>(clock::now() - t_setup).count());
            r.dof_steps = dof_steps;
            if (rep) *rep = r;
            throw Error(ATM_DIVERGED, "non-finite residual norm at iteration " + std::to_string(it));
        }
        if (v <= sol_.tol) {
            r.converged = 1;
            r.stop_reason = 0;
            status = ATM_OK;
            break;
        }
    }
    sync_stream(__func__);
    r.total_seconds = std::chrono::duration<double>(clock::now() - t0).count();
    host_phase("iterations", std::chrono::duration<double>(clock::now() - t_setup).count());
    r.dof_steps = dof_steps;
    if (rep) *rep = r;
    return status;
}

// ---------------------------------------------------------------------------
// state access and kernel-level entry points

// copy [first, first+count) of one array kind between host and device,
// one 2D copy per owning shard
void Engine::xfer_level(int level, int which, int first, int count, double* host, bool to_host) {
    if (level < 0 || level >= H_.L) config_error("level out of range");
    if (count < 0 || first < 0 || first + count > H_.np[level]) config_error("point range out of range");
    if (!to_host) {
        setup();
        relax_valid_ = halo0_valid_ = false;
    }
    if (level == 0) flush_guess();
    sync_stream(__func__);
    if (to_host && level == 0 && which == 0 && cpts_) {
        get_level0_cpts(first, count, host);
        return;
    }
    // one process sees every shard (world 1): every row is written below;
    // with one shard per process, points this process does not own read as 0
    if (to_host && world_ > 1) std::fill(host, host + static_cast<size_t>(count) * n_, 0.0);
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[level];
        DArr* a = which == 0 ? &Lv.u : which == 1 ? &Lv.g : which == 2 ? &Lv.v : &Lv.r;
        if (!a->p) continue;
        // owned points (plus, for writes, any allocated row such as halos);
        // with C-point storage (div > 1) writes reach only the held C points
        const int dv = a->div, top = a->base + (a->rows - 1) * dv;
        int lo = to_host ? std::max(Lv.lo, a->base) : a->base;
        int hi = to_host ? std::min(Lv.hi, top) : top;
        lo = std::max(lo, first);
        hi = std::min(hi, first + count - 1);
        if (hi < lo) continue;
        lo = a->base + (lo - a->base + dv - 1) / dv * dv;
        hi = a->base + (hi - a->base) / dv * dv;
        if (hi < lo) continue;
        const int nrow = (hi - lo) / dv + 1;
        double* h = host + static_cast<size_t>(lo - first) * n_;
        double* d = a->p + a->off(lo, pitch_);
        (to_host ? d2h_bytes_ : h2d_bytes_) += sizeof(double) * n_ * static_cast<size_t>(nrow);
        if (to_host)
            CK(cudaMemcpy2DAsync(h, sizeof(double) * n_ * dv, d, sizeof(double) * pitch_,
                                 sizeof(double) * n_, nrow, cudaMemcpyDeviceToHost, st_));
        else
            CK(cudaMemcpy2DAsync(d, sizeof(double) * pitch_, h, sizeof(double) * n_ * dv,
                                 sizeof(double) * n_, nrow, cudaMemcpyHostToDevice, st_));
    }
    sync_stream(__func__);
}

// Level-0 u with C-point storage: the requested points are rebuilt chunk by
// chunk of whole intervals -- the held C rows copied into a full-row scratch
// block whose F rows an F-sweep (STORE_ALL) recomputes -- then copied out.
// Scratch is bounded (~1 GiB), so any N_t can be read back.
void Engine::get_level0_cpts(int first, int count, double* out) {
    const int m = H_.m[0], last = H_.np[0] - 1;
    const size_t rowb = sizeof(double) * pitch_;
    if (world_ > 1) std::fill(out, out + static_cast<size_t>(count) * n_, 0.0);
    const int ivc = static_cast<int>(std::max<size_t>(1, (size_t(1) << 30) / (rowb * m)));
    for (Shard& s : sh_) {
        LevelDev& Lv = s.lv[0];
        const int lo = std::max(Lv.lo, first), hi = std::min(Lv.hi, first + count - 1);
        if (hi < lo) continue;
        const int nJ = hi / m - lo / m + 1;
        LevelDev tmp;
        DArr T = alloc_arr(tmp, 0, std::min(nJ, ivc) * m + 1, true, Lvl_[0]);
        for (int J0 = lo / m; J0 * m <= hi; J0 += ivc) {
            const int J1 = std::min(hi / m + 1, J0 + ivc);  // intervals [J0, J1)
            const int cb = J0 * m, ce = std::min(last, J1 * m - 1);
            T.base = cb;
            CK(cudaMemcpy2DAsync(T.p, rowb * m, Lv.u.p + Lv.u.off(cb, pitch_), rowb, rowb, J1 - J0,
                                 cudaMemcpyDeviceToDevice, st_));
            std::swap(Lv.u, T);
            try {
                sweep_jobs(s, 0, SW_F, J0, J1, TAIL_NONE, 0, nullptr, 0, STORE_ALL);
            } catch (...) {
                std::swap(Lv.u, T);
                throw;
            }
            std::swap(Lv.u, T);
            const int r0 = std::max(lo, cb), r1 = std::min(hi, ce);
            d2h_bytes_ += sizeof(double) * n_ * static_cast<size_t>(r1 - r0 + 1);
            CK(cudaMemcpy2DAsync(out + static_cast<size_t>(r0 - first) * n_, sizeof(double) * n_,
                                 T.p + T.off(r0, pitch_), rowb, sizeof(double) * n_, r1 - r0 + 1,
                                 cudaMemcpyDeviceToHost, st_));
        }
        sync_stream(__func__);
        for (void* p : tmp.allocs) cudaFree(p);
    }
    check_newton();
}

void Engine::get_level(int level, int which, int first, int count, double* out) {
    xfer_level(level, which, first, count, out, true);
}

void Engine::set_level(int level, int which, int first, int count, const double* in) {
    xfer_level(level, which, first, count, const_cast<double*>(in), false);
}

void Engine::apply_phi(int level, int first, int count, const double* in, double* out,
                       bool forcing) {
    if (level < 0 || level >= H_.L) config_error("level out of range");
    if (count <= 0) return;
    if (first < 1 || first + count > H_.np[level]) config_error("step index out of range");
    Shard& s = sh_[0];
    LevelDev tmp;
    DArr x = alloc_arr(tmp, 0, count, true);
    DArr y = alloc_arr(tmp, 0, count, true);
    if (!forcing)
        CK(cudaMemcpy2DAsync(x.p, sizeof(double) * pitch_, in, sizeof(double) * n_,
                             sizeof(double) * n_, count, cudaMemcpyHostToDevice, st_));
    const int forced = forcing ? 1 : (phi_forced_);
    LevelDev save = s.lv[level];
    if (!heat_ && !h2d_ && forcing) {
        // scalar forcing(level, i): ff[i] on level 0 explicit, else zero
        std::vector<double> h(count, 0.0);
        for (int j = 0; j < count; ++j) {
            const int i = first + j;
            h[j] = (!folded_ && level == 0 && i < static_cast<int>(ff_.size())) ? ff_[i] : 0.0;
        }
        std::memcpy(out, h.data(), sizeof(double) * count);
    } else {
        window_launch(s, level, WK_APPLY, 0, 0, -1, 0, count - 1, x, x, x, y, 1, forced,
                      forcing ? 1 : 0, first, 0);
        CK(cudaMemcpy2DAsync(out, sizeof(double) * n_, y.p, sizeof(double) * pitch_,
                             sizeof(double) * n_, count, cudaMemcpyDeviceToHost, st_));
    }
    sync_stream(__func__);
    (void)save;
    for (void* p : tmp.allocs) cudaFree(p);
    check_newton();
}

void Engine::kernel_f_relax(int level, int first_iv, int count) {
    if (level == 0 && cpts_)
        config_error("kernel-level entry points need full level-0 storage");
    relax_valid_ = halo0_valid_ = false;
    if (G_ != 1) config_error("kernel-level entry points need a single shard");
    setup();
    flush_guess();
    sweep_jobs(sh_[0], level, SW_F, first_iv, first_iv + count, TAIL_NONE, 0, nullptr, 0);
    sync_stream(__func__);
    check_newton();
}

void Engine::kernel_c_relax(int level, int first_c, int count) {
    if (level == 0 && cpts_)
        config_error("kernel-level entry points need full level-0 storage");
    relax_valid_ = halo0_valid_ = false;
    if (G_ != 1) config_error("kernel-level entry points need a single shard");
    setup();
    flush_guess();
    sweep_jobs(sh_[0], level, SW_CRELAX, std::max(1, first_c), first_c + count, TAIL_NONE, 0,
               nullptr, 0);
    sync_stream(__func__);
    check_newton();
}

void Engine::kernel_residual(int level, int first, int count, double* out) {
    if (level == 0 && cpts_)
        config_error("kernel-level entry points need full level-0 storage");
    if (G_ != 1) config_error("kernel-level entry points need a single shard");
    setup();
    flush_guess();
    Shard& s = sh_[0];
    LevelDev tmp;
    DArr r = alloc_arr(tmp, first, count, true, Lvl_.empty() ? 0 : Lvl_[level]);
    LevelDev& Lv = s.lv[level];
    if (heat_) {
        SweepArgs a{};
        a.co = Lv.hco;
        a.kind = SW_RESID;
        a.sq_div = 1;
        a.m = 1;
        a.np = H_.np[level];
        a.j0 = std::max(1, first);
        a.j1 = first + count;
        a.u_base = Lv.u.base;
        a.add_g = Lv.g_full;
        a.g_base = Lv.g_full ? Lv.g.base : 0;
        a.forced = phi_forced_;
        a.store = STORE_ALL;
        a.tail = TAIL_STORE;
        a.out_base = first;
        a.n_out = choose_n_out(a);
        const int grid = grid_for(a.j1 - a.j0, heat_sweep_occupancy(a));
        if (a.j1 > a.j0)
            check_launch(launch_heat_sweep(a, Lv.u.tm, Lv.g_full ? Lv.g.tm : Lv.u.tm, r.tm, Lv.u.tmw,
                                           r.tmw, grid, st_),
                         "resid");
    } else if (h2d_) {
        CgSweepArgs a{};
        a.co = Lv.gco;
        a.kind = SW_RESID;
        a.sq_div = 1;
        a.m = 1;
        a.np = H_.np[level];
        a.j0 = std::max(1, first);
        a.j1 = first + count;
        a.u = Lv.u.p;
        a.u_base = Lv.u.base;
        a.g = Lv.g_full ? Lv.g.p : nullptr;
        a.g_base = Lv.g_full ? Lv.g.base : 0;
        a.add_g = Lv.g_full;
        a.forced = phi_forced_;
        a.store = STORE_ALL;
        a.tail = TAIL_STORE;
        a.out = r.p;
        a.out_base = first;
        if (a.j1 > a.j0) check_launch(launch_cg_sweep(a, st_), "resid");
    } else {
        ScalarSweepArgs a{};
        a.co = Lv.sco;
        a.kind = SW_RESID;
        a.sq_div = 1;
        a.m = 1;
        a.np = H_.np[level];
        a.j0 = std::max(1, first);
        a.j1 = first + count;
        a.u = Lv.u.p;
        a.u_base = Lv.u.base;
        a.g = Lv.g_full ? Lv.g.p : nullptr;
        a.g_base = Lv.g_full ? Lv.g.base : 0;
        a.add_g = Lv.g_full;
        a.store = 1;
        a.tail = TAIL_STORE;
        a.out = r.p;
        a.out_base = first;
        check_launch(launch_scalar_sweep(a, st_), "resid");
    }
    if (first == 0 && Lv.g.p) check_launch(launch_row_diff(r.p, Lv.g.p, Lv.u.p, n_, nullptr, st_), "r0");
    CK(cudaMemcpy2DAsync(out, sizeof(double) * n_, r.p, sizeof(double) * pitch_, sizeof(double) * n_,
                         count, cudaMemcpyDeviceToHost, st_));
    sync_stream(__func__);
    for (void* p : tmp.allocs) cudaFree(p);
}

unsigned long long Engine::inner_iterations() {
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, d_inner_, sizeof(v), cudaMemcpyDeviceToHost, st_));
    sync_stream(__func__);
    return v;
}

int Engine::phase_times(char* names, int cap_names, double* secs, int cap, int* counts) const {
    // resolve pending events (const_cast: bookkeeping only)
    Engine* self = const_cast<Engine*>(this);
    if (!pending_.empty()) {
        cudaStreamSynchronize(st_);
        for (auto& pe : self->pending_) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, pe.second.first, pe.second.second) == cudaSuccess) {
                self->phase_sec_[pe.first] += ms * 1e-3;
                self->phase_cnt_[pe.first] += 1;
            }
            self->ev_pool_.push_back(pe.second.first);
            self->ev_pool_.push_back(pe.second.second);
        }
        self->pending_.clear();
    }
    std::string csv;
    int i = 0;
    for (const auto& kv : phase_sec_) {
        if (i >= cap) break;
        if (counts) {
            auto it = phase_cnt_.find(kv.first);
            counts[i] = it == phase_cnt_.end() ? 0 : it->second;
        }
        secs[i++] = kv.second;
        csv += (csv.empty() ? "" : ",") + kv.first;
    }
    if (names && cap_names > 0) {
        std::strncpy(names, csv.c_str(), cap_names - 1);
        names[cap_names - 1] = 0;
    }
    return i;
}

}  // namespace atm
