// heat2d_cg.cu -- 2D heat Phi chains for sm_100a (BASELINE configs 2, 4).
//
// Phi_i(u) = sub-steps of (I - dt Lap_h) x = u (+ dt f when folded), each
// solved by CG exactly as oracle/atm_oracle.c h2_solve restates it:
//   r = b - A x0 (x0 = u_prev), stop = rtol |b|, p = r;
//   while |r| > stop: ap = A p; alpha = rr / p.ap; x += alpha p;
//                     r -= alpha ap; beta = rr' / rr; p = r + beta p.
// A x = (1 + 4c) x - c (((x_w + x_e) + x_s) + x_n), c = dt / h^2.
//
// Layout: one system per thread-block cluster (cg_kernels.cuh).  p is kept
// in shared memory as (R + 2) x (nx + 2) doubles -- zero columns left and
// right, halo rows above/below copied from the neighbouring CTAs' shared
// memory through DSMEM after each cluster barrier -- so the stencil needs no
// bounds checks.  A p is recomputed in the update pass instead of stored.
//
// Job semantics (sweep: F / FCF / C-relax / residual with STORE or SQ
// tails; windows: linear / FAS / forward / apply / FAS right-hand side)
// are those of the scalar backend (common_kernels.cu) and the heat kernels,
// restating kernels.cpp:7-95 of the reference.
#include <cfloat>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <map>
#include <mutex>
#include <tuple>

#include "cg_kernels.cuh"
#include "heat_kernels.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace atm {

namespace {

constexpr int kMaxCgThreads = 1024;
constexpr size_t kCgSmemCap = 220 * 1024;

struct CgShared {
    double wred[32][2];      // per-warp partial sums
    double cslot[2][16][2];  // CTA partials of every cluster rank (parity double-buffered)
};

// per-CTA context
struct Ctx {
    int q, cs, rows, own, W, t, nt;
    int row0, col0, dq, dr;  // element k of thread t: idx = t + k nt -> (row, col)
    double* ps;              // (R + 2) x W, own rows 1..rows
    double* xs;              // own x (shared) or null
    double* rs;              // own r (shared) or null
    CgShared* sh;
    int par;
    double* ex;              // strip kernel: exchange area (strip_area_doubles)
    int spar;                // strip kernel: exchange parity
    uint32_t sph;            // strip kernel: mbarrier phase bit per parity
    unsigned long long gseq; // strip kernel, group mode: exchanges so far in this launch
};

__device__ __forceinline__ void csync(const Ctx& cx) {
    if (cx.cs > 1) cg::this_cluster().sync();
    else __syncthreads();
}

// fixed-order sum over the CTA, then over the cluster in rank order.  Thread
// 0 of every CTA writes its CTA partial into slot [rank] of every peer's
// shared memory (DSMEM stores) before the cluster barrier, so afterwards each
// thread sums cs local values (no per-thread DSMEM reads).
template <int NV>
__device__ __forceinline__ void cluster_sum(double (&v)[NV], Ctx& cx) {
    // local thread index: cx.t spans the whole cluster for Gray-Scott
    const int lt = threadIdx.x;
    const int lane = lt & 31, warp = lt >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) cx.sh->wred[warp][i] = v[i];
    __syncthreads();
    const int par = cx.par;
    cx.par ^= 1;
    if (cx.cs == 1) {
        if (lt == 0) {
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                double s = 0.0;
                for (int w = 0; w < nw; ++w) s += cx.sh->wred[w][i];
                cx.sh->cslot[par][0][i] = s;
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = cx.sh->cslot[par][0][i];
        return;
    }
    cg::cluster_group cl = cg::this_cluster();
    if (lt < cx.cs) {
        // thread r delivers this CTA's partials to peer r
        double part[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += cx.sh->wred[w][i];
            part[i] = s;
        }
        double* dst = cl.map_shared_rank(&cx.sh->cslot[par][cx.q][0], lt);
#pragma unroll
        for (int i = 0; i < NV; ++i) dst[i] = part[i];
    }
    cl.sync();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
        for (int r = 0; r < cx.cs; ++r) s += cx.sh->cslot[par][r][i];
        v[i] = s;
    }
}

// halo rows from the neighbouring CTAs (after a cluster barrier)
__device__ __forceinline__ void halos(const Ctx& cx, int nx, int R) {
    if (cx.cs == 1) return;
    cg::cluster_group cl = cg::this_cluster();
    const int W = cx.W;
    if (cx.q > 0) {
        const double* src = cl.map_shared_rank(cx.ps, cx.q - 1) + static_cast<size_t>(R) * W;
        for (int c = cx.t; c < nx; c += cx.nt) cx.ps[1 + c] = src[1 + c];
    }
    if (cx.q < cx.cs - 1) {
        const double* src = cl.map_shared_rank(cx.ps, cx.q + 1) + W;
        double* dst = cx.ps + static_cast<size_t>(cx.rows + 1) * W;
        for (int c = cx.t; c < nx; c += cx.nt) dst[1 + c] = src[1 + c];
    }
    __syncthreads();
}

// own-element iteration: f(idx, off), idx = t + j nt (coalesced, conflict-free)
template <class F>
__device__ __forceinline__ void for_own(const Ctx& cx, F&& f) {
    int row = cx.row0, col = cx.col0;
    const int nx = cx.W - 2;
#pragma unroll 2
    for (int idx = cx.t; idx < cx.own; idx += cx.nt) {
        f(idx, (row + 1) * cx.W + col + 1);
        col += cx.dr;
        row += cx.dq;
        if (col >= nx) {
            col -= nx;
            ++row;
        }
    }
}

__device__ __forceinline__ double stencil(const double* ps, int off, int W, double diag, double c) {
    return diag * ps[off] - c * (((ps[off - 1] + ps[off + 1]) + ps[off - W]) + ps[off + W]);
}

// Phi in place on the cluster's x (xb: this CTA's band of x; rb: its band
// of the residual r)
__device__ void cg_phi(const CgCoefDev& co, Ctx& cx, double* xb, double* rb, int band,
                       bool forced) {
    const int W = cx.W;
    const double c = co.c, diag = co.diag;
    for (int s = 0; s < co.substeps; ++s) {
        // prologue: p <- x0, r = b - A x0, |b|, |r|
        for_own(cx, [&](int idx, int off) { cx.ps[off] = xb[idx]; });
        csync(cx);
        halos(cx, co.nx, co.R);
        double v2[2] = {0.0, 0.0};
        for_own(cx, [&](int idx, int off) {
            double b = cx.ps[off];
            if (forced) b += co.sdt * __ldg(co.src + band + idx);
            const double rk = b - stencil(cx.ps, off, W, diag, c);
            rb[idx] = rk;
            v2[0] = fma(b, b, v2[0]);
            v2[1] = fma(rk, rk, v2[1]);
        });
        cluster_sum<2>(v2, cx);
        const double stop = co.rtol * sqrt(v2[0]);
        double rr = v2[1];
        for_own(cx, [&](int idx, int off) { cx.ps[off] = rb[idx]; });
        int it = 0;
        while (sqrt(rr) > stop) {
            if (it >= co.cg_max) {
                if (cx.t == 0 && cx.q == 0) atomicExch(co.fail, 1);
                break;
            }
            csync(cx);
            halos(cx, co.nx, co.R);
            double pap[1] = {0.0};
            for_own(cx, [&](int, int off) {
                pap[0] = fma(cx.ps[off], stencil(cx.ps, off, W, diag, c), pap[0]);
            });
            cluster_sum<1>(pap, cx);
            const double alpha = rr / pap[0];
            double rn[1] = {0.0};
            for_own(cx, [&](int idx, int off) {
                const double pk = cx.ps[off];
                const double ap = stencil(cx.ps, off, W, diag, c);
                xb[idx] += alpha * pk;
                const double rk = rb[idx] - alpha * ap;
                rb[idx] = rk;
                rn[0] = fma(rk, rk, rn[0]);
            });
            cluster_sum<1>(rn, cx);
            const double beta = rn[0] / rr;
            rr = rn[0];
            for_own(cx, [&](int idx, int off) { cx.ps[off] = rb[idx] + beta * cx.ps[off]; });
            ++it;
        }
        if (co.iters && cx.t == 0 && cx.q == 0) atomicAdd(co.iters, static_cast<unsigned long long>(it));
    }
}

// ---------------------------------------------------------------------------
// Strip kernel (systems up to nx = 255): one cluster barrier per CG iteration.
//
// The standard CG above needs three cluster-wide synchronisations per
// iteration (p halos, p.Ap, r.r) and streams p, x, r through shared memory
// for every stencil -- it is bound by shared-memory bandwidth and barrier
// latency, not by the FP64 pipe.  Here every vector lives in registers:
// lane l of warp (wx, wy) of cluster CTA q owns grid column wx*32 + l and the
// E consecutive rows q*R + wy*E + [0, E) (R = E * WY), so north/south
// neighbours are the thread's own registers and west/east ones are lane
// shuffles; only strip ends (one value per thread) and warp-edge columns (E
// values per warp) cross threads through shared memory / DSMEM.
//
// The iteration is Chronopoulos-Gear CG (same Krylov iterates as h2_solve's
// CG in exact arithmetic: alpha_i = gamma_i / (p_i, A p_i) with
// (p_i, A p_i) = delta_i - beta_i gamma_i / alpha_{i-1}):
//     x += alpha p;  r -= alpha s;  w = A r;  gamma = (r, r), delta = (w, r)
//     [one barrier: the two dots and w's boundary values]
//     stop if |r| <= rtol |b|;  beta = gamma / gamma_old;
//     alpha = gamma / (delta - beta gamma / alpha_old);  p = r + beta p;  s = w + beta s
// w = A r needs the neighbours' NEW r, which is only published after the
// next barrier; instead every thread MIRRORS its halo points' r and s with the
// same recurrences (r_h -= alpha s_h, s_h = w_h + beta s_h, explicit fma in
// both places), fed only by the neighbours' published w.  The mirror is
// therefore bitwise the neighbour's own value, and the stencil's inputs are
// complete after a single barrier.  Dot products: warp trees, then every warp
// pushes its two partials to every CTA of the cluster; after the barrier each
// warp sums the cs * NW partials in the same fixed order, so all threads hold
// bitwise the same alpha and beta (shard-count independent).
// 1 / a: MUFU.RCP64H seed refined by two Newton steps (full fp64 accuracy
// to a few ulp; no slow path -- the CG scalars are finite and nonzero)
__device__ __forceinline__ double rcp_nr(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    return fma(y, e, y);
}

template <int E>
struct Strip {
    int WX, WY, NW, C, cs, q, nx;
    int wx, wy, lane, warp, col;
    bool hasN, hasS, hasW, hasE;
    double *sN, *sS, *sW, *sE, *mir, *red;
    uint64_t* bar;       // two mbarriers (one per parity) counting peer CTAs' st.async bytes
    uint32_t rx_bytes;   // bytes this CTA receives from its peers per exchange
    int rcs, rq;         // dot-partial slots: [par][rcs][NW] (group mode: local, rcs = 1)
    // group mode: this group's global rows [par][cs][top | bottom][C],
    // CTA partials [par][cs] and sequence flags [cs]
    double* grows;
    double2* gred;
    unsigned long long* gflag;
    double *pbuf, *sbuf;  // group mode: p and s, [E][nt] each
};

__host__ __device__ inline size_t glob_doubles(int cs, int C) {
    return 2 * 2 * static_cast<size_t>(cs) * C + 2 * 2 * static_cast<size_t>(cs);
}

__host__ __device__ inline size_t strip_area_doubles(int WX, int WY, int E, int cs) {
    const size_t C = static_cast<size_t>(WX) * 32;
    return 2 * 2 * static_cast<size_t>(WY) * C          // N / S row slots, two parities
           + 2 * 2 * static_cast<size_t>(WY) * WX * E   // W / E column slots, two parities
           + 4 * static_cast<size_t>(WY) * WX * E       // reader-owned r / s mirrors of the W / E columns
           + 2 * static_cast<size_t>(cs) * WX * WY * 2  // dot partials, two parities
           + 2;                                         // two mbarriers
}

template <int E>
__device__ __forceinline__ Strip<E> strip_init(const CgCoefDev& co, const Ctx& cx, double* area) {
    Strip<E> S;
    S.WX = co.sWX;
    S.WY = co.sWY;
    S.NW = S.WX * S.WY;
    S.C = S.WX * 32;
    S.cs = cx.cs;
    S.q = cx.q;
    S.nx = co.nx;
    S.lane = threadIdx.x & 31;
    S.warp = threadIdx.x >> 5;
    S.wx = S.warp % S.WX;
    S.wy = S.warp / S.WX;
    S.col = S.wx * 32 + S.lane;
    S.hasN = S.wy > 0 || S.q > 0;
    S.hasS = S.wy + 1 < S.WY || S.q + 1 < S.cs;
    S.hasW = S.wx > 0;
    S.hasE = S.wx + 1 < S.WX;
    const size_t rowslots = 2 * static_cast<size_t>(S.WY) * S.C;
    const size_t colslots = 2 * static_cast<size_t>(S.WY) * S.WX * E;
    S.sN = area;
    S.sS = S.sN + rowslots;
    S.sW = S.sS + rowslots;
    S.sE = S.sW + colslots;
    S.mir = S.sE + colslots;
    S.red = S.mir + 2 * colslots;
    S.rcs = co.glob ? 1 : S.cs;
    S.rq = co.glob ? 0 : S.q;
    S.bar = reinterpret_cast<uint64_t*>(S.red + 2 * static_cast<size_t>(S.rcs) * S.NW * 2);
    S.rx_bytes = static_cast<uint32_t>((S.cs - 1) * S.NW * 16 + ((S.q > 0) + (S.q + 1 < S.cs)) * S.C * 8);
    S.grows = nullptr;
    S.gred = nullptr;
    S.gflag = nullptr;
    S.pbuf = S.sbuf = nullptr;
    if (co.glob) {
        const int group = blockIdx.x / S.cs;
        double* gb = co.gex + static_cast<size_t>(group) * glob_doubles(S.cs, S.C);
        S.grows = gb;
        S.gred = reinterpret_cast<double2*>(gb + 2 * 2 * static_cast<size_t>(S.cs) * S.C);
        S.gflag = co.gflag + static_cast<size_t>(group) * S.cs;
        S.pbuf = reinterpret_cast<double*>(S.bar + 2);
        S.sbuf = S.pbuf + static_cast<size_t>(E) * blockDim.x;
    }
    return S;
}

// once per kernel (strip geometry, cs > 1): the exchange mbarriers, visible
// to every peer before anyone sends
__device__ __forceinline__ void strip_bar_init(const CgCoefDev& co, double* area) {
    // slots and mirrors across the domain boundary are read but never written:
    // they must hold zeros
    {
        const size_t n = strip_area_doubles(co.sWX, co.sWY, co.E % 1000, co.glob ? 1 : co.cs) - 2;
        for (size_t i = threadIdx.x; i < n; i += blockDim.x) area[i] = 0.0;
        __syncthreads();
    }
    if (co.cs > 1 && !co.glob) {
        if (threadIdx.x == 0) {
            const int WX = co.sWX, WY = co.sWY, E = co.E % 1000;
            uint64_t* bar = reinterpret_cast<uint64_t*>(area + strip_area_doubles(WX, WY, E, co.cs) - 2);
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            mbar_fence_init();
        }
        cg::this_cluster().sync();
    }
}

// W / E column slot of warp (wx, wy) at parity par
template <int E>
__device__ __forceinline__ size_t strip_cslot(const Strip<E>& S, int par, int wx) {
    return ((static_cast<size_t>(par) * S.WY + S.wy) * S.WX + wx) * E;
}

// hand this thread's boundary values of v (and two dot partials) to the
// threads / CTAs that read them after the next barrier
template <int E, bool G>
__device__ __forceinline__ void strip_publish(const Strip<E>& S, int par, const double (&v)[E], double g0,
                                              double g1) {
    // peers' data arrive by st.async, counted on their mbarrier for this parity
    const uint32_t bar = smem_u32(S.bar + par);
    if (!G && S.cs > 1 && threadIdx.x == 0) mbar_expect_tx_u32(bar, S.rx_bytes);
    // bottom row -> the north slot of the warp-row below; top row -> the
    // south slot of the warp-row above (next / previous CTA across the band
    // edge: DSMEM st.async, or the group's global rows)
    if (S.wy + 1 < S.WY) {
        S.sN[(static_cast<size_t>(par) * S.WY + S.wy + 1) * S.C + S.col] = v[E - 1];
    } else if (G) {
        if (S.q + 1 < S.cs) __stcg(&S.grows[((static_cast<size_t>(par) * S.cs + S.q) * 2 + 1) * S.C + S.col], v[E - 1]);
    } else if (S.q + 1 < S.cs) {
        st_async_f64(mapa_u32(smem_u32(&S.sN[(static_cast<size_t>(par) * S.WY) * S.C + S.col]), S.q + 1), v[E - 1],
                     mapa_u32(bar, S.q + 1));
    }
    if (S.wy > 0) {
        S.sS[(static_cast<size_t>(par) * S.WY + S.wy - 1) * S.C + S.col] = v[0];
    } else if (G) {
        if (S.q > 0) __stcg(&S.grows[((static_cast<size_t>(par) * S.cs + S.q) * 2) * S.C + S.col], v[0]);
    } else if (S.q > 0) {
        st_async_f64(mapa_u32(smem_u32(&S.sS[(static_cast<size_t>(par) * S.WY + S.WY - 1) * S.C + S.col]), S.q - 1),
                     v[0], mapa_u32(bar, S.q - 1));
    }
    // east column -> west slot of the warp to the right; west column -> east
    // slot of the warp to the left
    if (S.lane == 31 && S.hasE) {
        double2* d = reinterpret_cast<double2*>(S.sW + strip_cslot(S, par, S.wx + 1));
#pragma unroll
        for (int k = 0; k < E; k += 2) d[k >> 1] = make_double2(v[k], v[k + 1]);
    }
    if (S.lane == 0 && S.hasW) {
        double2* d = reinterpret_cast<double2*>(S.sE + strip_cslot(S, par, S.wx - 1));
#pragma unroll
        for (int k = 0; k < E; k += 2) d[k >> 1] = make_double2(v[k], v[k + 1]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        g0 += __shfl_xor_sync(0xffffffffu, g0, off);
        g1 += __shfl_xor_sync(0xffffffffu, g1, off);
    }
    if (S.lane == 0) {
        const size_t at = ((static_cast<size_t>(par) * S.rcs + S.rq) * S.NW + S.warp) * 2;
        *reinterpret_cast<double2*>(&S.red[at]) = make_double2(g0, g1);
        if (!G) {
            const uint32_t a = smem_u32(&S.red[at]);
            for (int rk = 0; rk < S.cs; ++rk)
                if (rk != S.q) st_async_v2f64(mapa_u32(a, rk), g0, g1, mapa_u32(bar, rk));
        }
    }
}

__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// group mode exchange: the CTA's warp partials (local slots at parity par)
// summed in a fixed tree, published with the boundary rows (already stored)
// under this CTA's sequence flag; then wait for every CTA of the group.
// Cooperative launch: all CTAs of the grid are co-resident.
__device__ __forceinline__ void glob_sync(const double* red_local, int NW, double2* gred, unsigned long long* gflag,
                                          int cs, int q, int par, unsigned long long seq) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double a0 = 0.0, a1 = 0.0;
        if (lane < NW) {
            const double2 v = *reinterpret_cast<const double2*>(red_local + (static_cast<size_t>(par) * NW + lane) * 2);
            a0 = v.x;
            a1 = v.y;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, off);
            a1 += __shfl_xor_sync(0xffffffffu, a1, off);
        }
        if (lane == 0) {
            __stcg(&gred[static_cast<size_t>(par) * cs + q], make_double2(a0, a1));
            // one arrival on the group's counter, released at gpu scope:
            // cumulative over the CTA's row stores, ordered before it by the
            // barrier above; then wait for all cs arrivals of this exchange
            red_release_gpu_add_u64(&gflag[0], 1ull);
            const unsigned long long want = seq * static_cast<unsigned long long>(cs);
            while (ld_acquire_gpu_u64(&gflag[0]) < want) {
            }
        }
        __syncwarp();
    }
    __syncthreads();
}

// group mode: the cs CTA partials, in CTA order, xor tree (all lanes agree)
__device__ __forceinline__ void glob_dots(const double2* gred, int cs, int par, double& g0, double& g1) {
    const int lane = threadIdx.x & 31;
    double a0 = 0.0, a1 = 0.0;
    for (int i = lane; i < cs; i += 32) {
        const double2 v = __ldcg(&gred[static_cast<size_t>(par) * cs + i]);
        a0 += v.x;
        a1 += v.y;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, off);
        a1 += __shfl_xor_sync(0xffffffffu, a1, off);
    }
    g0 = a0;
    g1 = a1;
}

// the exchange's completion: local slots by the CTA barrier, peers' st.async
// data by this parity's mbarrier phase (no cluster-wide barrier: a CTA can run
// at most one exchange ahead of a peer, and each parity's buffers are reused
// only after every peer has consumed them -- they reply before moving on)
template <int E, bool G>
__device__ __forceinline__ void strip_sync(const Strip<E>& S, int par, uint32_t& phase, unsigned long long& seq) {
    if (G) {
        glob_sync(S.red, S.NW, S.gred, S.gflag, S.cs, S.q, par, ++seq);
        return;
    }
    __syncthreads();
    if (S.cs > 1) {
        mbar_wait_cluster(smem_u32(S.bar + par), (phase >> par) & 1u);
        phase ^= 1u << par;
    }
}

// the cluster's two dot products: the cs * NW warp partials summed in the
// same order by every warp of every CTA (lane-strided sums, then an xor tree:
// commutative pairings, so all lanes agree bitwise)
template <int E, bool G>
__device__ __forceinline__ void strip_dots(const Strip<E>& S, int par, double& g0, double& g1) {
    if (G) {
        glob_dots(S.gred, S.cs, par, g0, g1);
        return;
    }
    const int tot = S.cs * S.NW;
    const double* r = S.red + static_cast<size_t>(par) * tot * 2;
    double a0 = 0.0, a1 = 0.0;
    for (int i = S.lane; i < tot; i += 32) {
        const double2 v = *reinterpret_cast<const double2*>(r + 2 * i);
        a0 += v.x;
        a1 += v.y;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, off);
        a1 += __shfl_xor_sync(0xffffffffu, a1, off);
    }
    g0 = a0;
    g1 = a1;
}

// north / south values published for this thread at parity par (0 across
// the domain boundary)
template <int E, bool G>
__device__ __forceinline__ void strip_ns(const Strip<E>& S, int par, double& vn, double& vs) {
    // slots across the domain boundary are never written: they stay at the
    // zeros of strip_bar_init (Dirichlet)
    vn = S.sN[(static_cast<size_t>(par) * S.WY + S.wy) * S.C + S.col];
    vs = S.sS[(static_cast<size_t>(par) * S.WY + S.wy) * S.C + S.col];
    if (G) {
        if (S.wy == 0)
            vn = S.q > 0 ? __ldcg(&S.grows[((static_cast<size_t>(par) * S.cs + S.q - 1) * 2 + 1) * S.C + S.col]) : 0.0;
        if (S.wy + 1 == S.WY)
            vs = S.q + 1 < S.cs ? __ldcg(&S.grows[((static_cast<size_t>(par) * S.cs + S.q + 1) * 2) * S.C + S.col])
                                : 0.0;
    }
}

// out = A v on this thread's strip (zero outside the grid); hw / he: the W / E
// column values for lanes 0 / 31 (zeros across the domain boundary).  FULL:
// every point of the warp's strips is inside the grid (no masking).
template <int E, bool FULL>
__device__ __forceinline__ void strip_apply(const Strip<E>& S, const double (&v)[E], double vn, double vs,
                                            const double* hw, const double* he, const bool (&ok)[E],
                                            double diag, double c, double (&out)[E]) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
        // branch-free: every lane loads the (broadcast) halo pair, lanes 0 / 31 select it
        const double2 hw2 = reinterpret_cast<const double2*>(hw)[k >> 1];
        const double2 he2 = reinterpret_cast<const double2*>(he)[k >> 1];
        const double hwk = (k & 1) ? hw2.y : hw2.x, hek = (k & 1) ? he2.y : he2.x;
        double west = __shfl_up_sync(0xffffffffu, v[k], 1);
        double east = __shfl_down_sync(0xffffffffu, v[k], 1);
        west = S.lane == 0 ? hwk : west;
        east = S.lane == 31 ? hek : east;
        const double up = k > 0 ? v[k - 1] : vn;
        const double dn = k < E - 1 ? v[k + 1] : vs;
        // h2_apply's association: ((west + east) + row above) + row below
        const double a = diag * v[k] - c * (((west + east) + up) + dn);
        out[k] = (FULL || ok[k]) ? a : 0.0;
    }
}

template <int E>
__device__ __forceinline__ void strip_apply(const Strip<E>& S, bool full, const double (&v)[E], double vn,
                                            double vs, const double* hw, const double* he, const bool (&ok)[E],
                                            double diag, double c, double (&out)[E]) {
#ifdef ATM_STRIP_FULL_PATH
    if (full) strip_apply<E, true>(S, v, vn, vs, hw, he, ok, diag, c, out);
    else
#endif
    strip_apply<E, false>(S, v, vn, vs, hw, he, ok, diag, c, out);
}

template <int E, bool G>
__device__ void cg_phi_strip(const CgCoefDev& co, Ctx& cx, double* xb, int band, bool forced) {
    const Strip<E> S = strip_init<E>(co, cx, cx.ex);
    const double c = co.c, diag = co.diag;
    const int nx = co.nx;
    const int lrow0 = S.wy * E;
    uint32_t phase = cx.sph;
    unsigned long long seq = cx.gseq;
    bool ok[E];
#pragma unroll
    for (int k = 0; k < E; ++k) ok[k] = S.col < nx && lrow0 + k < cx.rows;
    // warp-uniform: no grid padding anywhere in this warp's strips
    const bool full = S.wx * 32 + 31 < nx && lrow0 + E <= cx.rows;
    const int base = lrow0 * nx + S.col;
    // reader-owned mirrors of the W / E halo columns: [rW | sW | rE | sE]
    const size_t mstride = static_cast<size_t>(S.WY) * S.WX * E;
    double* mrW = S.mir + (static_cast<size_t>(S.wy) * S.WX + S.wx) * E;
    double* msW = mrW + mstride;
    double* mrE = msW + mstride;
    double* msE = mrE + mstride;
    // mirror-update lanes: lanes [0, E) own W element `lane`, lanes [16, 16 + E) E element `lane - 16`
    const int mk = S.lane < 16 ? S.lane : S.lane - 16;
    const bool mlane = mk < E && (S.lane < 16 ? S.hasW : S.hasE);
    double* mr = S.lane < 16 ? mrW : mrE;
    double* ms = S.lane < 16 ? msW : msE;
    double* slotv = S.lane < 16 ? S.sW : S.sE;
    // group mode: x stays in the shared band xb, p and s in shared memory
    // [k][thread]; otherwise all CG vectors are registers
    double* const pg = S.pbuf + threadIdx.x;
    double* const sg = S.sbuf + threadIdx.x;
    const int nt = blockDim.x;

    __syncthreads();  // xb was written by the job code with its own thread map
    for (int sub = 0; sub < co.substeps; ++sub) {
        // xr: x (registers), or in group mode x0 for the prologue only
        double xr[E], r[E], w[E], p[G ? 1 : E], sv[G ? 1 : E];
#pragma unroll
        for (int k = 0; k < E; ++k) xr[k] = ok[k] ? xb[base + k * nx] : 0.0;
        // ---- r0 = b - A x0 (x0 = u_prev): x's boundary values first
        int par = cx.spar;
        strip_publish<E, G>(S, par, xr, 0.0, 0.0);
        strip_sync<E, G>(S, par, phase, seq);
        double xn, xs;
        strip_ns<E, G>(S, par, xn, xs);
        strip_apply(S, full, xr, xn, xs, S.sW + strip_cslot(S, par, S.wx), S.sE + strip_cslot(S, par, S.wx), ok, diag,
                    c, w);
        par ^= 1;
        double bb = 0.0, rr = 0.0;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            double b = xr[k];
            if (forced && ok[k]) b += co.sdt * __ldg(co.src + band + base + k * nx);
            r[k] = ok[k] ? b - w[k] : 0.0;
            bb = fma(b, b, bb);
            rr = fma(r[k], r[k], rr);
        }
        // ---- r0's boundary values, |b|^2 and |r0|^2
        strip_publish<E, G>(S, par, r, bb, rr);
        strip_sync<E, G>(S, par, phase, seq);
        strip_dots<E, G>(S, par, bb, rr);
        double rn, rs;
        strip_ns<E, G>(S, par, rn, rs);
        if (mlane) mr[mk] = slotv[strip_cslot(S, par, S.wx) + mk];
        __syncwarp();
        par ^= 1;
        const double stop = co.rtol * sqrt(bb);
        // h2_solve's test sqrt(rr) > stop without a square root on the
        // iteration's critical path: decided by rr against stop^2 with a
        // relative margin far above the rounding of either side, exact
        // sqrt only inside the margin
        const double stop2 = stop * stop, s2hi = stop2 * (1.0 + 1e-12), s2lo = stop2 * (1.0 - 1e-12);
        auto more = [&](double g) { return g > s2hi || (g >= s2lo && sqrt(g) > stop); };
        int it = 0;
        if (more(rr)) {
            // ---- w0 = A r0, delta0
            strip_apply(S, full, r, rn, rs, mrW, mrE, ok, diag, c, w);
            double delta = 0.0;
#pragma unroll
            for (int k = 0; k < E; ++k) delta = fma(w[k], r[k], delta);
            strip_publish<E, G>(S, par, w, delta, 0.0);
            strip_sync<E, G>(S, par, phase, seq);
            double dummy;
            strip_dots<E, G>(S, par, delta, dummy);
            double wn, ws;
            strip_ns<E, G>(S, par, wn, ws);
            double wh = mlane ? slotv[strip_cslot(S, par, S.wx) + mk] : 0.0;
            par ^= 1;
            double alpha = rr / delta, beta = 0.0;
            // 1 / gamma and 1 / alpha of the previous iteration, formed off the
            // critical path (one division per iteration remains on it)
            double rgamma = 1.0 / rr, ralpha = delta / rr;
            // p = s = 0 with beta = 0 makes the first update p0 = r0, s0 = w0
            double sn = 0.0, ss = 0.0;
            if (mlane) ms[mk] = 0.0;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                if constexpr (G) {
                    pg[k * nt] = 0.0;
                    sg[k * nt] = 0.0;
                } else {
                    p[k] = 0.0;
                    sv[k] = 0.0;
                }
            }
            bool go = co.cg_max > 0;
            if (!go && threadIdx.x == 0 && cx.q == 0) atomicExch(co.fail, 1);
#ifdef ATM_CG_PROF
            long long t_upd = 0, t_pub = 0, t_sync = 0, t_dots = 0, t0 = clock64();
#endif
            while (go) {
                // p = r + beta p, s = w + beta s, x += alpha p, r -= alpha s
                // (own points and mirrored halo points; explicit fma in both)
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    double pk, sk;
                    if constexpr (G) {
                        pk = fma(beta, pg[k * nt], r[k]);
                        sk = fma(beta, sg[k * nt], w[k]);
                        pg[k * nt] = pk;
                        sg[k * nt] = sk;
                        if (ok[k]) xb[base + k * nx] = fma(alpha, pk, xb[base + k * nx]);
                    } else {
                        pk = fma(beta, p[k], r[k]);
                        sk = fma(beta, sv[k], w[k]);
                        p[k] = pk;
                        sv[k] = sk;
                        xr[k] = fma(alpha, pk, xr[k]);
                    }
                    r[k] = fma(-alpha, sk, r[k]);
                }
                sn = fma(beta, sn, wn);
                ss = fma(beta, ss, ws);
                rn = fma(-alpha, sn, rn);
                rs = fma(-alpha, ss, rs);
                if (mlane) {
                    const double m = fma(beta, ms[mk], wh);
                    ms[mk] = m;
                    mr[mk] = fma(-alpha, m, mr[mk]);
                }
                __syncwarp();
                // w = A r, gamma = (r, r), delta = (w, r): one exchange
                double g = 0.0, d = 0.0;
                strip_apply(S, full, r, rn, rs, mrW, mrE, ok, diag, c, w);
                {
                    // four interleaved partial sums (short FMA chains), fixed order
                    double ga[4] = {0.0, 0.0, 0.0, 0.0}, da[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int k = 0; k < E; ++k) {
                        ga[k & 3] = fma(r[k], r[k], ga[k & 3]);
                        da[k & 3] = fma(w[k], r[k], da[k & 3]);
                    }
                    g = (ga[0] + ga[1]) + (ga[2] + ga[3]);
                    d = (da[0] + da[1]) + (da[2] + da[3]);
                }
#ifdef ATM_CG_PROF
                long long t1 = clock64();
                t_upd += t1 - t0;
#endif
                strip_publish<E, G>(S, par, w, g, d);
#ifdef ATM_CG_PROF
                long long t2 = clock64();
                t_pub += t2 - t1;
#endif
                strip_sync<E, G>(S, par, phase, seq);
#ifdef ATM_CG_PROF
                long long t3 = clock64();
                t_sync += t3 - t2;
#endif
                strip_dots<E, G>(S, par, g, d);
                strip_ns<E, G>(S, par, wn, ws);
                wh = mlane ? slotv[strip_cslot(S, par, S.wx) + mk] : 0.0;
#ifdef ATM_CG_PROF
                t0 = clock64();
                t_dots += t0 - t3;
#endif
                par ^= 1;
                ++it;
                if (!more(g)) break;
                if (it >= co.cg_max) {
                    if (threadIdx.x == 0 && cx.q == 0) atomicExch(co.fail, 1);
                    break;
                }
                beta = g * rgamma;
                const double den = d - beta * g * ralpha;
                // alpha = g / den through a refined reciprocal (two Newton
                // steps from the hardware seed: a few ulp, identical in every
                // thread of the group) instead of the IEEE division sequence
                const double rden = rcp_nr(den);
                alpha = g * rden;
                rgamma = rcp_nr(g);
                ralpha = den * rgamma;
            }
#ifdef ATM_CG_PROF
            if ((threadIdx.x == 0 || threadIdx.x == 200) && blockIdx.x < 2 && it > 0)
                printf("cgprof blk %d thr %d it %d upd %lld pub %lld sync %lld dots %lld (cycles/it)\n", blockIdx.x,
                       threadIdx.x, it, t_upd / it, t_pub / it, t_sync / it, t_dots / it);
#endif
        }
        cx.spar = par;
        cx.sph = phase;
        cx.gseq = seq;
        if (co.iters && threadIdx.x == 0 && cx.q == 0) atomicAdd(co.iters, static_cast<unsigned long long>(it));
        if constexpr (!G) {
#pragma unroll
            for (int k = 0; k < E; ++k)
                if (ok[k]) xb[base + k * nx] = xr[k];
        }
    }
    __syncthreads();  // the job code reads xb with its own thread map
}

// group mode: the sum of one value over the group's CTAs (the sweep tails'
// C-point squares), through the same exchange as the CG dots
template <int E>
__device__ double group_sum1(const CgCoefDev& co, Ctx& cx, double v) {
    const Strip<E> S = strip_init<E>(co, cx, cx.ex);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int par = cx.spar;
    if (S.lane == 0) *reinterpret_cast<double2*>(&S.red[(static_cast<size_t>(par) * S.NW + S.warp) * 2]) =
        make_double2(v, 0.0);
    glob_sync(S.red, S.NW, S.gred, S.gflag, S.cs, S.q, par, ++cx.gseq);
    double g0, g1;
    glob_dots(S.gred, S.cs, par, g0, g1);
    cx.spar = par ^ 1;
    return g0;
}

// ---------------------------------------------------------------------------
// Gray-Scott Phi (gray_scott.cpp:91-190): backward Euler sub-steps, Newton
// on F(w) = w - w_prev - dt f(w) with stop = max(tol, tol |F_0|), the
// Jacobian J = I - dt f'(w) applied matrix-free, J delta = F by BiCGSTAB with
// diagonal (Jacobi) right preconditioning from delta = 0 to |r|^2 <= tol^2
// |F|^2 within 2 dim iterations (restart when rho degenerates) -- the
// published algorithm behind the reference's Eigen::BiCGSTAB, restated in
// oracle/atm_oracle.c gs_bicgstab; then the bounds check of step().  One CTA
// per system; w and the nine work vectors live in shared memory when they
// fit (n <= 36), else in ten global scratch rows per resident CTA (the
// paper's 128^2 grid: 2.6 MB per system, L2/HBM-streamed); CTA reductions in
// a fixed order either way.

struct GsVec {
    double *w, *prev, *x, *r, *r0, *p, *v, *s, *t, *yz;
};

__device__ __forceinline__ void gs_nbrs(int idx, int n, int cells, int& base, int& c, int& N,
                                        int& S, int& E, int& W) {
    base = idx >= cells ? cells : 0;
    c = idx - base;
    const int i = c / n, j = c - (c / n) * n;
    N = ((i + 1 == n) ? 0 : i + 1) * n + j;
    S = ((i == 0) ? n - 1 : i - 1) * n + j;
    E = i * n + ((j + 1 == n) ? 0 : j + 1);
    W = i * n + ((j == 0) ? n - 1 : j - 1);
}

// diagonal of J at element idx
__device__ __forceinline__ double gs_diag(const CgCoefDev& co, const double* w, int idx, int cells,
                                          double dt) {
    const int c = idx >= cells ? idx - cells : idx;
    const double u = w[c], v = w[cells + c];
    if (idx < cells) {
        double d = 1.0 + dt * 4.0 * co.gs_du * co.gs_h2inv;
        if (co.gs_reaction) d += dt * (v * v + co.gs_feed);
        return d;
    }
    double d = 1.0 + dt * 4.0 * co.gs_dv * co.gs_h2inv;
    if (co.gs_reaction) d += dt * (co.gs_feed + co.gs_kill) - dt * 2.0 * u * v;
    return d;
}

// (J x)[idx]
__device__ __forceinline__ double gs_jx(const CgCoefDev& co, const double* w, const double* x,
                                        int idx, int n, int cells, double dt) {
    int base, c, N, S, E, W;
    gs_nbrs(idx, n, cells, base, c, N, S, E, W);
    const double u = w[c], v = w[cells + c];
    const double nb = x[base + N] + x[base + S] + x[base + E] + x[base + W];
    if (idx < cells) {
        const double off = -dt * co.gs_du * co.gs_h2inv;
        double r = gs_diag(co, w, idx, cells, dt) * x[idx] + off * nb;
        if (co.gs_reaction) r += dt * 2.0 * u * v * x[cells + c];
        return r;
    }
    const double offv = -dt * co.gs_dv * co.gs_h2inv;
    double r = gs_diag(co, w, idx, cells, dt) * x[idx] + offv * nb;
    if (co.gs_reaction) r += -dt * v * v * x[c];
    return r;
}

// F[idx] = w - prev - dt f(w) (reaction_terms, gray_scott.cpp:63-88)
__device__ __forceinline__ double gs_res(const CgCoefDev& co, const double* w, const double* prev,
                                         int idx, int n, int cells, double dt) {
    int base, c, N, S, E, W;
    gs_nbrs(idx, n, cells, base, c, N, S, E, W);
    const double u = w[c], v = w[cells + c];
    const double lap = (w[base + N] + w[base + S] + w[base + E] + w[base + W] - 4.0 * w[idx]) * co.gs_h2inv;
    double f;
    if (idx < cells) {
        f = co.gs_du * lap;
        if (co.gs_reaction) f += -u * v * v + co.gs_feed * (1.0 - u);
    } else {
        f = co.gs_dv * lap;
        if (co.gs_reaction) f += u * v * v - (co.gs_feed + co.gs_kill) * v;
    }
    return w[idx] - prev[idx] - dt * f;
}

__device__ void gs_phi(const CgCoefDev& co, Ctx& cx, const GsVec& g) {
    const int n = co.nx, cells = n * n, m = 2 * cells;
    const double dt = co.sdt;
    auto loop = [&](auto&& f) {
        for (int idx = cx.t; idx < m; idx += cx.nt) f(idx);
    };
    bool failed = false;
    for (int sub = 0; sub < co.substeps && !failed; ++sub) {
        loop([&](int i) { g.prev[i] = g.w[i]; });
        csync(cx);
        double nr[1] = {0.0};
        loop([&](int i) {
            const double F = gs_res(co, g.w, g.prev, i, n, cells, dt);
            g.r[i] = F;
            nr[0] = fma(F, F, nr[0]);
        });
        cluster_sum<1>(nr, cx);
        const double norm0 = sqrt(nr[0]);
        const double stop = fmax(co.newton_tol, co.newton_tol * norm0);
        if (norm0 <= stop) continue;
        bool ok = false;
        for (int it = 0; it < co.newton_max; ++it) {
            // ---- BiCGSTAB: J x = b (b = F in r), x0 = 0
            double bb[1] = {0.0};
            loop([&](int i) {
                const double b = g.r[i];
                g.r0[i] = b;
                g.x[i] = 0.0;
                g.p[i] = 0.0;
                g.v[i] = 0.0;
                bb[0] = fma(b, b, bb[0]);
            });
            cluster_sum<1>(bb, cx);
            const double tol2 = co.gs_linear_tol * co.gs_linear_tol * bb[0];
            double rr = bb[0], r0n = bb[0];
            double rho = 1.0, alpha = 1.0, om = 1.0;
            const int maxit = 2 * m;
            int lit = 0, restarts = 0, done_it = 0;
            while (rr > tol2 && lit < maxit) {
                const double rho_old = rho;
                double d1[1] = {0.0};
                loop([&](int i) { d1[0] = fma(g.r0[i], g.r[i], d1[0]); });
                cluster_sum<1>(d1, cx);
                rho = d1[0];
                if (fabs(rho) < DBL_EPSILON * DBL_EPSILON * r0n) {  // Eigen BiCGSTAB restart rule
                    loop([&](int i) { g.r0[i] = g.r[i]; });
                    rho = r0n = rr;
                    if (restarts++ == 0) lit = 0;
                }
                const double beta = (rho / rho_old) * (alpha / om);
                loop([&](int i) {
                    const double pi = g.r[i] + beta * (g.p[i] - om * g.v[i]);
                    g.p[i] = pi;
                    g.yz[i] = pi / gs_diag(co, g.w, i, cells, dt);
                });
                csync(cx);
                double d2[1] = {0.0};
                loop([&](int i) {
                    const double vi = gs_jx(co, g.w, g.yz, i, n, cells, dt);
                    g.v[i] = vi;
                    d2[0] = fma(g.r0[i], vi, d2[0]);
                });
                cluster_sum<1>(d2, cx);
                alpha = rho / d2[0];
                loop([&](int i) {
                    g.x[i] += alpha * g.yz[i];
                    const double si = g.r[i] - alpha * g.v[i];
                    g.s[i] = si;
                });
                csync(cx);
                loop([&](int i) { g.yz[i] = g.s[i] / gs_diag(co, g.w, i, cells, dt); });
                csync(cx);
                double d3[2] = {0.0, 0.0};
                loop([&](int i) {
                    const double ti = gs_jx(co, g.w, g.yz, i, n, cells, dt);
                    g.t[i] = ti;
                    d3[0] = fma(ti, ti, d3[0]);
                    d3[1] = fma(ti, g.s[i], d3[1]);
                });
                cluster_sum<2>(d3, cx);
                om = d3[0] > 0.0 ? d3[1] / d3[0] : 0.0;
                double d4[1] = {0.0};
                loop([&](int i) {
                    g.x[i] += om * g.yz[i];
                    const double ri = g.s[i] - om * g.t[i];
                    g.r[i] = ri;
                    d4[0] = fma(ri, ri, d4[0]);
                });
                cluster_sum<1>(d4, cx);
                rr = d4[0];
                ++lit;
                ++done_it;
            }
            if (co.iters && cx.t == 0) atomicAdd(co.iters, static_cast<unsigned long long>(done_it));
            if (!(rr <= tol2)) break;  // inner linear solve failed
            // ---- Newton update and residual
            loop([&](int i) { g.w[i] -= g.x[i]; });
            csync(cx);
            double nn[1] = {0.0};
            loop([&](int i) {
                const double F = gs_res(co, g.w, g.prev, i, n, cells, dt);
                g.r[i] = F;
                nn[0] = fma(F, F, nn[0]);
            });
            cluster_sum<1>(nn, cx);
            if (sqrt(nn[0]) <= stop) {
                ok = true;
                break;
            }
        }
        if (!ok) failed = true;
    }
    if (failed) {
        if (cx.t == 0) atomicExch(co.fail, 1);
    } else if (co.gs_bounds_check) {
        bool bad = false;
        loop([&](int i) { bad = bad || !(g.w[i] >= co.gs_bound_lo && g.w[i] <= co.gs_bound_hi); });
        if (bad) atomicExch(co.fail, 2);
    }
    csync(cx);
}

template <int E>
__device__ __forceinline__ void cg_phi_any(const CgCoefDev& co, Ctx& cx, double* xb, double* rb,
                                           int band, bool forced) {
    if constexpr (E < 0) {
        // Gray-Scott: xb is vector 0 of the CTA's ten state-size vectors
        const int m = 2 * co.nx * co.nx;
        GsVec g{xb, xb + m, xb + 2 * m, xb + 3 * m, xb + 4 * m, xb + 5 * m, xb + 6 * m, xb + 7 * m,
                xb + 8 * m, xb + 9 * m};
        gs_phi(co, cx, g);
    } else if constexpr (E >= 3000) {
        cg_phi_strip<E % 1000, true>(co, cx, xb, band, forced);
    } else if constexpr (E >= 1000) {
        cg_phi_strip<E % 1000, false>(co, cx, xb, band, forced);
    } else {
        cg_phi(co, cx, xb, rb, band, forced);
    }
}

__device__ __forceinline__ void ctx_init(Ctx& cx, const CgCoefDev& co, unsigned char* smem) {
    cx.cs = co.cs;
    cx.q = co.glob ? static_cast<int>(blockIdx.x % co.cs)
                   : (co.cs > 1) ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
    cx.rows = max(0, min(co.R, co.nx - cx.q * co.R));
    cx.own = cx.rows * co.nx;
    cx.t = threadIdx.x;
    cx.nt = blockDim.x;
    if (co.prob == 1) {
        // Gray-Scott: the whole [u; v] state is the cluster's; its CTAs act
        // as one block of cs * nt threads over vectors in global scratch
        cx.rows = 2 * co.nx;
        cx.own = 2 * co.nx * co.nx;
        cx.t = cx.q * blockDim.x + threadIdx.x;
        cx.nt = co.cs * blockDim.x;
    }
    cx.W = co.nx + 2;
    cx.row0 = cx.t / co.nx;
    cx.col0 = cx.t - cx.row0 * co.nx;
    cx.dq = cx.nt / co.nx;
    cx.dr = cx.nt - cx.dq * co.nx;
    cx.sh = reinterpret_cast<CgShared*>(smem);
    cx.ps = reinterpret_cast<double*>(smem + sizeof(CgShared));
    const size_t psn = (co.prob == 1 || co.strip) ? 0 : static_cast<size_t>(co.R + 2) * cx.W;
    cx.xs = co.x_smem ? cx.ps + psn : nullptr;
    cx.rs = (co.x_smem && !co.strip) ? cx.ps + psn + static_cast<size_t>(co.R) * co.nx : nullptr;
    cx.ex = co.strip ? cx.ps + static_cast<size_t>(co.R) * co.nx : nullptr;
    cx.par = 0;
    cx.spar = 0;
    cx.sph = 0;
    cx.gseq = 0;
    // zero p (padding columns and the domain-boundary halo rows stay zero)
    for (size_t i = threadIdx.x; i < psn; i += blockDim.x) cx.ps[i] = 0.0;
    __syncthreads();
    if (co.strip) strip_bar_init(co, cx.ex);
}

// this CTA's band of the cluster's x and r (shared, or two global scratch
// rows per cluster slot)
__device__ __forceinline__ double* x_band(const CgCoefDev& co, const Ctx& cx, int slot) {
    if (co.prob == 1 && !co.x_smem) return co.xg + static_cast<size_t>(10 * slot) * co.pitch;
    return co.x_smem ? cx.xs
                     : co.xg + static_cast<size_t>(2 * slot) * co.pitch + static_cast<size_t>(cx.q) * co.R * co.nx;
}
__device__ __forceinline__ double* r_band(const CgCoefDev& co, const Ctx& cx, int slot) {
    return co.x_smem ? cx.rs
                     : co.xg + static_cast<size_t>(2 * slot + 1) * co.pitch + static_cast<size_t>(cx.q) * co.R * co.nx;
}

template <int E>
__global__ void __launch_bounds__(E >= 3000 ? 512 : E >= 2000 ? 256 : E > 0 ? 512 : kMaxCgThreads, 1) cg_sweep_kernel(const __grid_constant__ CgSweepArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx cx;
    ctx_init(cx, a.co, smem);
    const int cid = blockIdx.x / a.co.cs, ncl = gridDim.x / a.co.cs;
    const int band = a.co.prob == 1 ? 0 : cx.q * a.co.R * a.co.nx;
    double* xb = x_band(a.co, cx, cid);
    double* rb = r_band(a.co, cx, cid);
    const size_t P = a.co.pitch;
    auto row = [&](double* base, int i, int b0) { return base + static_cast<size_t>(i - b0) * P + band; };
    auto crow = [&](const double* base, int i, int b0) {
        return base + static_cast<size_t>(i - b0) * P + band;
    };
    const int m = a.m, last = a.np - 1;
    const int ud = a.u_div > 1 ? a.u_div : 1;
    for (int J = a.j0 + cid; J < a.j1; J += ncl) {
        const int c = J * m;
        int start, end, store_from;
        switch (a.kind) {
            case SW_FCF:
                start = (J == 0) ? 0 : c - m;
                store_from = (J == 0) ? 1 : c;
                end = min(c + m - 1, last);
                break;
            case SW_CRELAX: start = c - 1; end = c; store_from = c; break;
            case SW_RESID: start = c - 1; end = c - 1; store_from = INT_MAX; break;
            default: start = c; end = min(c + m - 1, last); store_from = c + 1; break;
        }
        if (end < start) end = start;
        {
            const double* src = crow(a.u, a.u_base + (start - a.u_base) / ud, a.u_base);
            for_own(cx, [&](int idx, int) { xb[idx] = src[idx]; });
        }
        for (int i = start + 1; i <= end; ++i) {
            cg_phi_any<E>(a.co, cx, xb, rb, band, a.forced);
            if (a.add_g) {
                const double* g = crow(a.g, i, a.g_base);
                for_own(cx, [&](int idx, int) { xb[idx] += g[idx]; });
            }
            if (i >= store_from && store_row(a.store, i, m)) {
                double* dst = row(a.u, i, a.u_base);
                for_own(cx, [&](int idx, int) { dst[idx] = xb[idx]; });
            }
        }
        if (a.tail != TAIL_NONE && end + 1 <= last && ((end + 1) % m) == 0) {
            const int ti = end + 1;
            cg_phi_any<E>(a.co, cx, xb, rb, band, a.forced);
            const double* g = a.add_g ? crow(a.g, ti, a.g_base) : nullptr;
            const double* uc = crow(a.u, a.u_base + (ti - a.u_base) / ud, a.u_base);
            if (a.tail == TAIL_STORE || a.tail == TAIL_BOTH) {
                double* dst = row(a.out, ti / m, a.out_base);
                for_own(cx, [&](int idx, int) {
                    double v = xb[idx];
                    if (g) v += g[idx];
                    dst[idx] = v - uc[idx];
                });
            }
            if (a.tail == TAIL_SQ || a.tail == TAIL_BOTH) {
                double s2[1] = {0.0};
                for_own(cx, [&](int idx, int) {
                    double v = xb[idx];
                    if (g) v += g[idx];
                    v -= uc[idx];
                    s2[0] = fma(v, v, s2[0]);
                });
                if constexpr (E >= 3000) s2[0] = group_sum1<E % 1000>(a.co, cx, s2[0]);
                else cluster_sum<1>(s2, cx);
                if (cx.q == 0 && cx.t == 0) a.sq[(ti - a.sq_base) / a.sq_div] = s2[0];
            }
        }
    }
    // no CTA may leave while a peer can still read its shared memory (DSMEM)
    if (a.co.cs > 1 && !a.co.glob) cg::this_cluster().sync();
}

template <int E>
__global__ void __launch_bounds__(E >= 3000 ? 512 : E >= 2000 ? 256 : E > 0 ? 512 : kMaxCgThreads, 1) cg_window_kernel(const __grid_constant__ CgWindowArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    Ctx cx;
    ctx_init(cx, a.co, smem);
    const int cid = blockIdx.x / a.co.cs, ncl = gridDim.x / a.co.cs;
    const int band = a.co.prob == 1 ? 0 : cx.q * a.co.R * a.co.nx;
    double* xb = x_band(a.co, cx, cid);
    double* rb = r_band(a.co, cx, cid);
    const size_t P = a.co.pitch;
    auto crow = [&](const double* base, int i, int b0) {
        return base + static_cast<size_t>(i - b0) * P + band;
    };
    auto orow = [&](int i) { return a.out + static_cast<size_t>(i - a.out_base) * P + band; };
    if (a.kind == WK_APPLY || a.kind == WK_FAS_RHS) {
        for (int p = a.p0 + cid; p <= a.p1; p += ncl) {
            if (a.kind == WK_APPLY) {
                if (a.seed_zero) {
                    for_own(cx, [&](int idx, int) { xb[idx] = 0.0; });
                } else {
                    const double* s = crow(a.x1, p + a.seed_off, a.x1_base);
                    for_own(cx, [&](int idx, int) { xb[idx] = s[idx]; });
                }
                cg_phi_any<E>(a.co, cx, xb, rb, band, a.forced);
                double* d = orow(p);
                for_own(cx, [&](int idx, int) { d[idx] = xb[idx]; });
            } else {
                // g_p = v_p - Psi(v_{p-1}) + r_p (solver.cpp:206-216)
                const double* s = crow(a.x1, p - 1, a.x1_base);
                for_own(cx, [&](int idx, int) { xb[idx] = s[idx]; });
                cg_phi_any<E>(a.co, cx, xb, rb, band, a.forced);
                const double* v = crow(a.x2, p, a.x2_base);
                const double* rr = crow(a.x3, p, a.x3_base);
                double* d = orow(p);
                for_own(cx, [&](int idx, int) {
                    double y = v[idx];
                    y -= xb[idx];
                    y += rr[idx];
                    d[idx] = y;
                });
            }
        }
        if (a.co.cs > 1 && !a.co.glob) cg::this_cluster().sync();
        return;
    }
    const bool has_pre = a.pre_e1 >= a.pre_e0;
    const int nj = (has_pre ? 1 : 0) + max(0, a.p1 - a.p0 + 1);
    for (int qj = cid; qj < nj; qj += ncl) {
        int lo, e0, e1;
        if (has_pre && qj == 0) {
            lo = a.pre_lo;
            e0 = a.pre_e0;
            e1 = a.pre_e1;
        } else {
            const int p = a.p0 + qj - (has_pre ? 1 : 0);
            lo = max(0, p - a.k + 1);
            e0 = e1 = p;
        }
        {
            const double* s1 = crow(a.x1, lo, a.x1_base);
            if (a.kind == WK_FAS) {
                const double* s2 = crow(a.x2, lo, a.x2_base);
                for_own(cx, [&](int idx, int) { xb[idx] = s2[idx] + s1[idx]; });
            } else {
                for_own(cx, [&](int idx, int) { xb[idx] = s1[idx]; });
            }
        }
        auto emit = [&](int p) {
            if (a.kind == WK_LINEAR) {
                double* d = a.out + static_cast<size_t>(p * a.out_stride - a.out_base) * P + band;
                for_own(cx, [&](int idx, int) { d[idx] += xb[idx]; });
            } else {
                double* d = orow(p);
                for_own(cx, [&](int idx, int) { d[idx] = xb[idx]; });
            }
        };
        if (lo >= e0) emit(lo);
        for (int s = lo + 1; s <= e1; ++s) {
            cg_phi_any<E>(a.co, cx, xb, rb, band, a.forced);
            if (a.kind == WK_LINEAR) {
                const double* r1 = crow(a.x1, s, a.x1_base);
                for_own(cx, [&](int idx, int) { xb[idx] += r1[idx]; });
            } else if (a.kind == WK_FAS) {
                const double* v = crow(a.x2, s, a.x2_base);
                const double* w = crow(a.x3, s, a.x3_base);
                const double* r1 = crow(a.x1, s, a.x1_base);
                for_own(cx, [&](int idx, int) {
                    double y = xb[idx];
                    y += v[idx];
                    y -= w[idx];
                    y += r1[idx];
                    xb[idx] = y;
                });
            }
            if (s >= e0) emit(s);
        }
    }
    if (a.co.cs > 1 && !a.co.glob) cg::this_cluster().sync();
}

struct CgKernels {
    const void* sweep;
    const void* window;
};

template <int E>
CgKernels cg_k() {
    return {reinterpret_cast<const void*>(cg_sweep_kernel<E>),
            reinterpret_cast<const void*>(cg_window_kernel<E>)};
}

// E = 0: round-1 cluster CG (p in shared memory, x and r shared or global);
// E = -1: Gray-Scott; 1000 + e / 2000 + e: strip kernel (512 / 256 threads);
// 3000 + e: strip kernel, group mode
CgKernels cg_kernels(int E) {
    switch (E) {
        case -1: return cg_k<-1>();
        case 1002: return cg_k<1002>();
        case 1004: return cg_k<1004>();
        case 2008: return cg_k<2008>();
        case 2012: return cg_k<2012>();
        case 2016: return cg_k<2016>();
        case 3008: return cg_k<3008>();
        case 3010: return cg_k<3010>();
        case 3012: return cg_k<3012>();
        case 3014: return cg_k<3014>();
        case 3016: return cg_k<3016>();
        default: return cg_k<0>();
    }
}

void cg_prepare(const void* fn) {
    static std::mutex mu;
    static std::map<const void*, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done[fn]) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done[fn] = true;
}

int cg_launch(const void* fn, const CgCoefDev& co, int jobs, void** args, cudaStream_t s) {
    if (jobs <= 0) return 0;
    cg_prepare(fn);
    const int ncl = std::min(jobs, cg_max_clusters(co));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncl * co.cs);
    cfg.blockDim = dim3(co.nt);
    cfg.dynamicSmemBytes = cg_smem_bytes(co);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (co.glob) {
        // group mode: every CTA of a group spins on its peers' flags, so the
        // whole grid must be co-resident (cooperative launch); flags restart
        // at zero for every launch
        const cudaError_t e = cudaMemsetAsync(co.gflag, 0, sizeof(unsigned long long) * ncl * co.cs, s);
        if (e != cudaSuccess) return static_cast<int>(e);
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    } else {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = co.cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelExC(&cfg, fn, args));
}

}  // namespace

// strip kernel geometry: WX warps across (32 columns each), WY warp-rows of
// E grid rows per CTA (R = E WY), cs = ceil(nx / R) CTAs per cluster (<= 16),
// at most 512 threads per CTA (5 E doubles of CG state per thread in
// registers); false when nx needs more than 16 CTAs of this shape
static bool strip_geometry(int nx, CgCoefDev& co) {
    if (const char* e = std::getenv("ATM_CG_STRIP"))
        if (std::atoi(e) == 0) return false;
    const int WX = (nx + 31) / 32;
    if (WX > 16) return false;
    // E >= 8: 256-thread CTAs (up to 255 registers: 5 E doubles of CG state
    // per thread plus the stencil's temporaries); E < 8: 512-thread CTAs
    int Es[5] = {16, 12, 8, 4, 2};
    if (const char* e = std::getenv("ATM_CG_STRIP_E")) Es[0] = Es[1] = Es[2] = Es[3] = Es[4] = std::atoi(e);
    for (int E : Es) {
        const int maxt = E >= 8 ? 256 : 512;
        if (32 * WX > maxt) continue;
        int WY = std::min(maxt / (32 * WX), (nx + E - 1) / E);
        if (const char* e = std::getenv("ATM_CG_STRIP_WY")) WY = std::min(WY, std::atoi(e));
        if (WY < 1) continue;
        const int R = E * WY;
        const int cs = (nx + R - 1) / R;
        if (cs > 16) continue;
        co.strip = 1;
        co.sWX = WX;
        co.sWY = WY;
        co.cs = cs;
        co.R = R;
        co.x_smem = 1;
        co.E = (E >= 8 ? 2000 : 1000) + E;
        co.nt = 32 * WX * WY;
        co.glob = 0;
        return true;
    }
    // group mode: one warp-row of WX warps per CTA (E grid rows), cs = G CTAs
    // of a cooperative grid per system; x, r, w in registers, p and s in
    // shared memory, exchanges through global memory
    if (const char* e = std::getenv("ATM_CG_GROUP"))
        if (std::atoi(e) == 0) return false;
    int Eg[5] = {14, 12, 16, 10, 8};
    if (const char* e = std::getenv("ATM_CG_STRIP_E")) Eg[0] = Eg[1] = Eg[2] = Eg[3] = Eg[4] = std::atoi(e);
    for (int E : Eg) {
        const int WY = 1;
        const int R = E * WY;
        const int G = (nx + R - 1) / R;
        co.strip = 1;
        co.glob = 1;
        co.sWX = WX;
        co.sWY = WY;
        co.cs = G;
        co.R = R;
        co.x_smem = 1;
        co.E = 3000 + E;
        co.nt = 32 * WX * WY;
        if (cg_smem_bytes(co) <= kCgSmemCap) return true;
    }
    co.strip = 0;
    co.glob = 0;
    return false;
}

void cg_geometry(int nx, CgCoefDev& co) {
    co.nx = nx;
    co.n = nx * nx;
    co.strip = 0;
    if (strip_geometry(nx, co)) return;
    const size_t red = sizeof(CgShared) + 64;
    // smallest cluster holding p, x and r on chip (up to 4 CTAs); else the
    // smallest cluster holding p, with x and r in global scratch rows
    int pick_cs = -1, pick_sm = 0;
    const char* force = std::getenv("ATM_CG_CS");  // tuning experiments
    for (int pass = 0; pass < 2 && pick_cs < 0; ++pass) {
        for (int cs = force ? std::atoi(force) : 1; cs <= 16; ++cs) {
            const int R = (nx + cs - 1) / cs;
            if ((cs - 1) * R >= nx) continue;
            const size_t ps = static_cast<size_t>(R + 2) * (nx + 2) * 8;
            const size_t xr = 2 * static_cast<size_t>(R) * nx * 8;
            if (pass == 0 && cs <= 4 && ps + xr + red <= kCgSmemCap) {
                pick_cs = cs;
                pick_sm = 1;
                break;
            }
            if (pass == 1 && ps + red <= kCgSmemCap) {
                pick_cs = cs;
                pick_sm = 0;
                break;
            }
        }
    }
    if (pick_cs < 0) {
        co.cs = 0;
        return;
    }
    co.cs = pick_cs;
    co.R = (nx + pick_cs - 1) / pick_cs;
    co.x_smem = pick_sm;
    const int own = co.R * nx;
    co.E = 0;
    co.nt = std::min(kMaxCgThreads, std::max(64, (own + 31) / 32 * 32));
}

bool gs_geometry(int nx, CgCoefDev& co, int cs) {
    co.nx = nx;
    co.n = 2 * nx * nx;
    co.prob = 1;
    co.cs = 1;
    co.R = 2 * nx;
    co.E = -1;
    co.x_smem = 1;
    co.nt = std::min(kMaxCgThreads, std::max(64, (co.n + 31) / 32 * 32));
    if (cg_smem_bytes(co) > kCgSmemCap) {
        co.x_smem = 0;  // work vectors in global scratch, shared by a cluster of cs CTAs
        co.cs = std::max(1, std::min(8, cs));
    }
    return true;
}

size_t cg_glob_doubles_per_group(const CgCoefDev& co) {
    return co.glob ? glob_doubles(co.cs, co.sWX * 32) : 0;
}

size_t cg_smem_bytes(const CgCoefDev& co) {
    if (co.prob == 1) return sizeof(CgShared) + (co.x_smem ? 10 * static_cast<size_t>(co.n) * 8 : 0);
    if (co.strip)
        return sizeof(CgShared) + static_cast<size_t>(co.R) * co.nx * 8 +
               strip_area_doubles(co.sWX, co.sWY, co.E % 1000, co.glob ? 1 : co.cs) * 8 +
               (co.glob ? 2 * static_cast<size_t>(co.E % 1000) * co.nt * 8 : 0);
    size_t b = sizeof(CgShared) + static_cast<size_t>(co.R + 2) * (co.nx + 2) * 8;
    if (co.x_smem) b += 2 * static_cast<size_t>(co.R) * co.nx * 8;
    return b;
}

int cg_max_clusters(const CgCoefDev& co) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, size_t>, int> cache;
    const size_t smem = cg_smem_bytes(co);
    const auto key = std::make_tuple(co.E, co.cs, co.nt, smem);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const void* fn = cg_kernels(co.E).sweep;
    cg_prepare(fn);
    cg_prepare(cg_kernels(co.E).window);
    if (co.glob) {
        // groups of cs co-resident CTAs (both kernels share the geometry)
        int per_sm = 0, per_sm_w = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, co.nt, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, cg_kernels(co.E).window, co.nt, smem);
        const int n = std::max(1, std::min(per_sm, per_sm_w) * sms / co.cs);
        if (std::getenv("ATM_DEBUG_OCC"))
            std::fprintf(stderr, "cg groups: G %d nt %d smem %zu per_sm %d/%d -> %d\n", co.cs, co.nt, smem, per_sm,
                         per_sm_w, n);
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = n;
        return n;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(co.cs * 148);
    cfg.blockDim = dim3(co.nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = co.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, fn, &cfg);
    if (std::getenv("ATM_DEBUG_OCC"))
        std::fprintf(stderr, "cg clusters: cs %d nt %d smem %zu -> %d (%s)\n", co.cs, co.nt, smem, n,
                     cudaGetErrorString(e));
    if (e != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = 1;
    }
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = n;
    return n;
}

int launch_cg_sweep(const CgSweepArgs& a, cudaStream_t s) {
    CgSweepArgs aa = a;
    void* args[] = {&aa};
    return cg_launch(cg_kernels(a.co.E).sweep, a.co, a.j1 - a.j0, args, s);
}

int launch_cg_window(const CgWindowArgs& a, cudaStream_t s) {
    int nj;
    if (a.kind == WK_APPLY || a.kind == WK_FAS_RHS) nj = a.p1 - a.p0 + 1;
    else nj = ((a.pre_e1 >= a.pre_e0) ? 1 : 0) + std::max(0, a.p1 - a.p0 + 1);
    CgWindowArgs aa = a;
    void* args[] = {&aa};
    return cg_launch(cg_kernels(a.co.E).window, a.co, nj, args, s);
}

}  // namespace atm
