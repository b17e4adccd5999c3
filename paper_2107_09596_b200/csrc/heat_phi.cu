// heat_phi.cu -- Heat1D Phi chains for sm_100a.
//
// One CTA owns one state vector (a time point) in registers, blocked
// (thread t holds elements [t*L, t*L+L)).  Rows move HBM <-> smem by TMA
// (cp.async.bulk.tensor, 128B-swizzled so the blocked register view reads
// and writes smem conflict-free); produced rows leave through TMA-store
// staging so stores overlap the next Phi.  The kernels are persistent: each
// CTA walks a contiguous range of jobs, so the row that closes job J (the
// residual's C-point) is the seed of job J+1 and is loaded once.
//
// Reference semantics restated (file:line under /root/reference/proj):
//   Phi / step          heat1d.cpp:47-60 (Thomas), :66-83 (sub-steps, forcing)
//   F-relaxation        kernels.cpp:7-17      -> SW_F jobs
//   C-relaxation        kernels.cpp:19-28     -> SW_CRELAX jobs / fused SW_FCF
//   residual / restrict kernels.cpp:30-43, solver.cpp:174-185 -> tails, SW_RESID
//   window solves       kernels.cpp:53-88     -> heat_window_*_kernel
//   point squares       kernels.cpp:90-95     -> TAIL_SQ (fixed-order tree)
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "heat_kernels.cuh"
#include "tma.cuh"

namespace atm {

// --------------------------------------------------------------------------
// host: coefficients and scan / carry multipliers

HeatLevelHost heat_level_host(int n, int pitch, int L, double sub_dt, double h, int substeps) {
    HeatLevelHost H;
    H.n = n;
    H.pitch = pitch;
    H.L = L;
    H.substeps = substeps;
    const int nt = (((pitch + L - 1) / L) + 31) / 32 * 32;
    H.nt = nt;
    const int npad = nt * L;
    // heat1d.cpp:28-44: r = sub_dt/h^2, a = -r, b = 1 + 2r, den_i = b - a c'_{i-1}
    H.r = sub_dt / (h * h);
    const double a = -H.r;
    const double b = 1.0 + 2.0 * H.r;
    std::vector<double> beta(npad, 0.0), cpr(npad, 0.0);
    double prev_c = 0.0;
    for (int i = 0; i < n; ++i) {
        const double den = b - a * prev_c;
        beta[i] = 1.0 / den;
        prev_c = a / den;
        cpr[i] = prev_c;
    }
    H.beta.assign(npad, 0.0);
    H.gamma.assign(npad, 0.0);
    H.cneg.assign(npad, 0.0);
    for (int i = 0; i < n; ++i) {
        H.beta[i] = beta[i];
        H.gamma[i] = H.r * beta[i];
        // the backward sweep never reads c'_{n-1} (heat1d.cpp:56)
        H.cneg[i] = (i == n - 1) ? 0.0 : -cpr[i];
    }
    // converged tail: the c' recurrence is a contraction; past i0 the
    // coefficients agree with their limit to <= 2 ulp and live in registers
    H.i0 = ((n + L - 1) / L) * L;
    if (n >= 3) {
        const double bc = beta[n - 2], cc = -cpr[n - 2];
        auto close = [](double x, double y) { return std::fabs(x - y) <= 4.5e-16 * std::fabs(y); };
        int last_diff = -1;
        for (int i = 0; i < n - 1; ++i)
            if (!close(beta[i], bc) || !close(-cpr[i], cc)) last_diff = i;
        H.i0 = ((last_diff + 1 + L - 1) / L) * L;
        H.beta_c = bc;
        H.gamma_c = H.r * bc;
        H.cneg_c = cc;
    }
    // effective per-element coefficients exactly as the device uses them
    std::vector<double> eg(npad), ec(npad);
    for (int t = 0; t < nt; ++t) {
        const int s = t * L;
        const bool cst = (s >= H.i0) && (s + L <= n - 1);
        for (int e = 0; e < L; ++e) {
            eg[s + e] = cst ? H.gamma_c : H.gamma[s + e];
            ec[s + e] = cst ? H.cneg_c : H.cneg[s + e];
        }
    }
    // per-thread fix-up products and chunk products
    H.pf.assign(npad, 0.0);
    H.pb.assign(npad, 0.0);
    std::vector<double> Af(nt), Ab(nt);
    for (int t = 0; t < nt; ++t) {
        double p = 1.0;
        for (int e = 0; e < L; ++e) {
            p *= eg[t * L + e];
            H.pf[t * L + e] = p;
        }
        Af[t] = p;
        p = 1.0;
        for (int e = L - 1; e >= 0; --e) {
            p *= ec[t * L + e];
            H.pb[t * L + e] = p;
        }
        Ab[t] = p;
    }
    H.powc.assign(2 * kMaxL, 0.0);
    {
        double p = 1.0;
        for (int e = 0; e < L; ++e) {
            p *= H.gamma_c;
            H.powc[e] = p;
        }
        p = 1.0;
        for (int e = L - 1; e >= 0; --e) {
            p *= H.cneg_c;
            H.powc[kMaxL + e] = p;
        }
    }
    // warp scan multipliers (Hillis-Steele over lanes) and warp products
    H.scan.assign(static_cast<size_t>(nt) * kScanPerThread, 0.0);
    const int nw = nt / 32;
    std::vector<double> AWf(nw), AWb(nw);
    for (int w = 0; w < nw; ++w) {
        double pf = 1.0, pb = 1.0;
        for (int l = 0; l < 32; ++l) pf *= Af[32 * w + l];
        for (int l = 31; l >= 0; --l) pb *= Ab[32 * w + l];
        AWf[w] = pf;
        AWb[w] = pb;
        for (int l = 0; l < 32; ++l) {
            double* sc = &H.scan[static_cast<size_t>(32 * w + l) * kScanPerThread];
            for (int d = 0; d < 5; ++d) {
                const int off = 1 << d;
                double mf = 0.0, mb = 0.0;
                if (l >= off) {
                    mf = 1.0;
                    for (int u = l - off + 1; u <= l; ++u) mf *= Af[32 * w + u];
                }
                if (l + off <= 31) {
                    mb = 1.0;
                    for (int u = l; u <= l + off - 1; ++u) mb *= Ab[32 * w + u];
                }
                sc[d] = mf;
                sc[6 + d] = mb;
            }
            double ex = 1.0;
            for (int u = 0; u < l; ++u) ex *= Af[32 * w + u];
            sc[5] = ex;
            double exb = 1.0;
            for (int u = l + 1; u <= 31; ++u) exb *= Ab[32 * w + u];
            sc[11] = exb;
        }
    }
    // cross-warp carry weights: carry_w = sum_{v<w} (prod_{u=v+1}^{w-1} AWf_u) T_v
    H.wf.assign(kMaxWarps * kMaxWarps, 0.0);
    H.wb.assign(kMaxWarps * kMaxWarps, 0.0);
    for (int w = 0; w < nw; ++w) {
        for (int v = 0; v < w; ++v) {
            double p = 1.0;
            for (int u = v + 1; u <= w - 1; ++u) p *= AWf[u];
            H.wf[w * kMaxWarps + v] = p;
        }
        for (int v = w + 1; v < nw; ++v) {
            double p = 1.0;
            for (int u = w + 1; u <= v - 1; ++u) p *= AWb[u];
            H.wb[w * kMaxWarps + v] = p;
        }
    }
    return H;
}

// --------------------------------------------------------------------------
// device: per-thread state, shared tables and the tridiagonal solve

template <int L>
struct Lane {
    int t, lane, warp, nw, s;
    bool cst;
    double Mf[5], Pfex, Mb[5], Pbex;
};

template <int L>
__device__ __forceinline__ void lane_init(Lane<L>& ln, const HeatCoefDev& co) {
    ln.t = threadIdx.x;
    ln.lane = ln.t & 31;
    ln.warp = ln.t >> 5;
    ln.nw = blockDim.x >> 5;
    ln.s = ln.t * L;
    ln.cst = (ln.s >= co.i0) && (ln.s + L <= co.n - 1);
    const double* sc = co.scan + ln.t * kScanPerThread;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        ln.Mf[d] = __ldg(sc + d);
        ln.Mb[d] = __ldg(sc + 6 + d);
    }
    ln.Pfex = __ldg(sc + 5);
    ln.Pbex = __ldg(sc + 11);
}

struct Tabs {              // per-CTA copy of the level's small tables
    double wf[kMaxWarps * kMaxWarps];
    double wb[kMaxWarps * kMaxWarps];
    double powc[2 * kMaxL];
};

struct Slots {             // small shared scratch
    double swf[kMaxWarps];
    double swb[kMaxWarps];
    double red[kMaxWarps];
    uint64_t bar[4];
};

__device__ __forceinline__ void tabs_init(Tabs& tb, const HeatCoefDev& co) {
    for (int i = threadIdx.x; i < kMaxWarps * kMaxWarps; i += blockDim.x) {
        tb.wf[i] = co.wf[i];
        tb.wb[i] = co.wb[i];
    }
    for (int i = threadIdx.x; i < 2 * kMaxL; i += blockDim.x) tb.powc[i] = co.powc[i];
}

// (I + sub_dt L) x = x, in place, over the CTA (heat1d.cpp:47-60).
template <int L>
__device__ __forceinline__ void tri_solve(double (&x)[L], const HeatCoefDev& co,
                                          const Lane<L>& ln, const Tabs& tb, Slots& sl) {
    // forward  y_i = beta_i x_i + gamma_i y_{i-1}   (local: zero carry-in)
    double y = 0.0;
    if (ln.cst) {
        const double bb = co.beta_c, gg = co.gamma_c;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            y = fma(gg, y, bb * x[e]);
            x[e] = y;
        }
    } else {
        const double* bt = co.beta + ln.s;
        const double* gt = co.gamma + ln.s;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            y = fma(__ldg(gt + e), y, __ldg(bt + e) * x[e]);
            x[e] = y;
        }
    }
    double B = y;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const double o = __shfl_up_sync(0xffffffffu, B, 1 << d);
        if (ln.lane >= (1 << d)) B = fma(ln.Mf[d], o, B);
    }
    double ex = __shfl_up_sync(0xffffffffu, B, 1);
    if (ln.lane == 0) ex = 0.0;
    if (ln.lane == 31) sl.swf[ln.warp] = B;
    __syncthreads();
    {
        const double* wr = tb.wf + ln.warp * kMaxWarps;
        double c0 = 0.0, c1 = 0.0;
        int v = 0;
        for (; v + 1 < ln.warp; v += 2) {
            c0 = fma(wr[v], sl.swf[v], c0);
            c1 = fma(wr[v + 1], sl.swf[v + 1], c1);
        }
        if (v < ln.warp) c0 = fma(wr[v], sl.swf[v], c0);
        const double carry = fma(ln.Pfex, c0 + c1, ex);
        if (ln.cst) {
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(carry, tb.powc[e], x[e]);
        } else {
            const double* pt = co.pf + ln.s;
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(carry, __ldg(pt + e), x[e]);
        }
    }
    // backward  x_i = y_i - c'_i x_{i+1}   (local: zero carry-in)
    double z = 0.0;
    if (ln.cst) {
        const double cc = co.cneg_c;
#pragma unroll
        for (int e = L - 1; e >= 0; --e) {
            z = fma(cc, z, x[e]);
            x[e] = z;
        }
    } else {
        const double* ct = co.cneg + ln.s;
#pragma unroll
        for (int e = L - 1; e >= 0; --e) {
            z = fma(__ldg(ct + e), z, x[e]);
            x[e] = z;
        }
    }
    B = z;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const double o = __shfl_down_sync(0xffffffffu, B, 1 << d);
        if (ln.lane + (1 << d) <= 31) B = fma(ln.Mb[d], o, B);
    }
    ex = __shfl_down_sync(0xffffffffu, B, 1);
    if (ln.lane == 31) ex = 0.0;
    if (ln.lane == 0) sl.swb[ln.warp] = B;
    __syncthreads();
    {
        const double* wr = tb.wb + ln.warp * kMaxWarps;
        double c0 = 0.0, c1 = 0.0;
        int v = ln.warp + 1;
        for (; v + 1 < ln.nw; v += 2) {
            c0 = fma(wr[v], sl.swb[v], c0);
            c1 = fma(wr[v + 1], sl.swb[v + 1], c1);
        }
        if (v < ln.nw) c0 = fma(wr[v], sl.swb[v], c0);
        const double carry = fma(ln.Pbex, c0 + c1, ex);
        if (ln.cst) {
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(carry, tb.powc[kMaxL + e], x[e]);
        } else {
            const double* pt = co.pb + ln.s;
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(carry, __ldg(pt + e), x[e]);
        }
    }
}

// Phi_index on this level: S sub-steps, forcing added before each solve
// when `forced` (heat1d.cpp:66-83).
template <int L>
__device__ __forceinline__ void phi(double (&x)[L], const HeatCoefDev& co, const Lane<L>& ln,
                                    const Tabs& tb, Slots& sl, int index, int forced) {
    for (int s = 0; s < co.substeps; ++s) {
        if (forced) {
            const double th = __ldg(co.theta + static_cast<size_t>(index) * co.substeps + s);
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(th, __ldg(co.prof + ln.s + e), x[e]);
        }
        tri_solve<L>(x, co, ln, tb, sl);
    }
}

// --------------------------------------------------------------------------
// device: swizzled row staging (TMA SWIZZLE_128B layout)

__device__ __forceinline__ int swz(int e) {
    const int q = e >> 4, ch = (e & 15) >> 1;
    return (q << 7) + ((ch ^ (q & 7)) << 4);
}

template <int L>
__device__ __forceinline__ void row_load(const char* buf, double (&x)[L], int s, int pitch) {
#pragma unroll
    for (int c = 0; c < L / 2; ++c) {
        const int e = s + 2 * c;
        if (e < pitch) {
            const double2 v = *reinterpret_cast<const double2*>(buf + swz(e));
            x[2 * c] = v.x;
            x[2 * c + 1] = v.y;
        } else {
            x[2 * c] = 0.0;
            x[2 * c + 1] = 0.0;
        }
    }
}

template <int L>
__device__ __forceinline__ void row_store(char* buf, const double (&x)[L], int s, int pitch) {
#pragma unroll
    for (int c = 0; c < L / 2; ++c) {
        const int e = s + 2 * c;
        if (e < pitch) *reinterpret_cast<double2*>(buf + swz(e)) = make_double2(x[2 * c], x[2 * c + 1]);
    }
}

// x = x + row, or x = x - row
template <int L>
__device__ __forceinline__ void row_acc(const char* buf, double (&x)[L], int s, int pitch,
                                        bool sub) {
#pragma unroll
    for (int c = 0; c < L / 2; ++c) {
        const int e = s + 2 * c;
        if (e < pitch) {
            const double2 v = *reinterpret_cast<const double2*>(buf + swz(e));
            if (sub) {
                x[2 * c] -= v.x;
                x[2 * c + 1] -= v.y;
            } else {
                x[2 * c] += v.x;
                x[2 * c + 1] += v.y;
            }
        }
    }
}

// fixed-order CTA reduction of sum x_e^2 (thread order, then warp xor tree,
// then warps in order): depends only on the CTA shape
template <int L>
__device__ __forceinline__ double cta_sum_squares(const double (&x)[L], const Lane<L>& ln,
                                                  Slots& sl) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < L; ++e) s = fma(x[e], x[e], s);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (ln.lane == 0) sl.red[ln.warp] = s;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < ln.nw; ++w) tot += sl.red[w];
    return tot;
}

__device__ __forceinline__ char* align1k(unsigned char* p) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__host__ __device__ inline int row_bytes_al(int pitch) { return ((pitch * 8) + 1023) & ~1023; }

// --------------------------------------------------------------------------
// sweep kernel: F / fused FCF / C-relax / residual jobs over C-point indices
// smem: [S seed/tail][O0][O1 if n_out=2][A if add_g][Tabs][Slots]

template <int L, int NTMAX, int MINB>
__global__ void __launch_bounds__(NTMAX, MINB)
    heat_sweep_kernel(const __grid_constant__ SweepArgs a, const __grid_constant__ CUtensorMap tm_u,
                      const __grid_constant__ CUtensorMap tm_g,
                      const __grid_constant__ CUtensorMap tm_out) {
    extern __shared__ unsigned char smem_raw[];
    char* base = align1k(smem_raw);
    const int pitch = a.co.pitch;
    const int rb = row_bytes_al(pitch);
    const int nob = a.n_out;
    char* bufS = base;
    char* bufO[2] = {base + rb, base + (nob == 2 ? 2 : 1) * rb};
    char* bufA = base + (1 + nob) * rb;
    char* tl = base + (1 + nob + (a.add_g ? 1 : 0)) * rb;
    Tabs& tb = *reinterpret_cast<Tabs*>(tl);
    Slots& sl = *reinterpret_cast<Slots*>(tl + sizeof(Tabs));
    uint64_t* barS = &sl.bar[0];
    uint64_t* barA = &sl.bar[1];
    const uint32_t bytes = static_cast<uint32_t>(pitch * 8);
    const int R = pitch >> 4;

    Lane<L> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    tabs_init(tb, a.co);
    if (t == 0) {
        mbar_init(barS, 1);
        mbar_init(barA, 1);
        mbar_fence_init();
        prefetch_tmap(&tm_u);
    }
    __syncthreads();
    uint32_t phS = 0, phA = 0;
    int ob = 0;

    const long long Nj = a.j1 - a.j0;
    const int jb = a.j0 + static_cast<int>(Nj * blockIdx.x / gridDim.x);
    const int je = a.j0 + static_cast<int>(Nj * (blockIdx.x + 1) / gridDim.x);
    const int m = a.m, last = a.np - 1;
    bool seed_ready = false;
    double x[L];

    // stage x into an output buffer and TMA-store it; the store that last
    // read that buffer was waited for (bulk_wait_read) before the Phi
    auto stage_out = [&](int row, const CUtensorMap* map) {
        char* o = bufO[ob];
        row_store<L>(o, x, ln.s, pitch);
        fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            tma_store_2d(map, 0, row * R, o);
            bulk_commit();
        }
        ob = (nob == 2) ? ob ^ 1 : 0;
    };

    for (int J = jb; J < je; ++J) {
        const int c = J * m;
        int start, end, store_from;
        switch (a.kind) {
            case SW_FCF:
                start = (J == 0) ? 0 : c - m;
                store_from = (J == 0) ? 1 : c;
                end = min(c + m - 1, last);
                break;
            case SW_CRELAX:
                start = c - 1;
                end = c;
                store_from = c;
                break;
            case SW_RESID:
                start = c - 1;
                end = c - 1;
                store_from = INT_MAX;
                break;
            default:  // SW_F
                start = c;
                end = min(c + m - 1, last);
                store_from = c + 1;
                break;
        }
        if (end < start) end = start;
        const int tail_i =
            (a.tail != TAIL_NONE && end + 1 <= last && ((end + 1) % m) == 0) ? end + 1 : -1;

        // ---- seed row
        if (!seed_ready) {
            if (t == 0) {
                mbar_expect_tx(barS, bytes);
                tma_load_2d(bufS, &tm_u, 0, (start - a.u_base) * R, barS);
            }
            mbar_wait(barS, phS);
            phS ^= 1;
        }
        row_load<L>(bufS, x, ln.s, pitch);
        // WAR across proxies: our generic reads of S must be ordered before
        // the TMA (async proxy) write that refills it
        fence_proxy_async();
        __syncthreads();
        seed_ready = false;
        if (tail_i >= 0 && t == 0) {
            mbar_expect_tx(barS, bytes);
            tma_load_2d(bufS, &tm_u, 0, (tail_i - a.u_base) * R, barS);
        }

        // ---- chain steps u_i = Phi_i(u_{i-1}) (+ g_i)
        for (int i = start + 1; i <= end; ++i) {
            if (a.add_g && t == 0) {
                mbar_expect_tx(barA, bytes);
                tma_load_2d(bufA, &tm_g, 0, (i - a.g_base) * R, barA);
            }
            if (t == 0) {
                if (nob == 2) bulk_wait_read<1>();
                else bulk_wait_read<0>();
            }
            phi<L>(x, a.co, ln, tb, sl, i, a.forced);
            if (a.add_g) {
                mbar_wait(barA, phA);
                phA ^= 1;
                row_acc<L>(bufA, x, ln.s, pitch, false);
            }
            if (a.store && i >= store_from) {
                stage_out(i - a.u_base, &tm_u);
            } else if (a.add_g) {
                fence_proxy_async();
                __syncthreads();  // bufA consumed before the next load
            }
        }

        // ---- tail: residual at the next C-point, r = Phi(u_last) + g_c - u_c
        if (tail_i >= 0) {
            if (a.add_g && t == 0) {
                mbar_expect_tx(barA, bytes);
                tma_load_2d(bufA, &tm_g, 0, (tail_i - a.g_base) * R, barA);
            }
            if (t == 0) {
                if (nob == 2) bulk_wait_read<1>();
                else bulk_wait_read<0>();
            }
            phi<L>(x, a.co, ln, tb, sl, tail_i, a.forced);
            if (a.add_g) {
                mbar_wait(barA, phA);
                phA ^= 1;
                row_acc<L>(bufA, x, ln.s, pitch, false);
            }
            mbar_wait(barS, phS);
            phS ^= 1;
            row_acc<L>(bufS, x, ln.s, pitch, true);
            if (a.kind == SW_F && J + 1 < je) seed_ready = true;  // S holds u[c_{J+1}]
            if (a.tail == TAIL_STORE) {
                stage_out(tail_i / m - a.out_base, &tm_out);
            } else {
                const double tot = cta_sum_squares<L>(x, ln, sl);
                if (t == 0) a.sq[tail_i - a.sq_base] = tot;
            }
        }
    }
    if (t == 0) bulk_wait<0>();
}

// --------------------------------------------------------------------------
// linear window kernel (kernels.cpp:53-61 + solver.cpp:271-278):
// e = r_lo, e = Psi_s(e) + r_s, fine u[c_p] += e.  The r rows of every job of
// the CTA form one stream, double-buffered two rows ahead; the fine C-point
// row is fetched into S ahead of its emit, updated in place and stored back.
// smem: [A0][A1][S][Tabs][Slots]

template <int L, int NTMAX, int MINB>
__global__ void __launch_bounds__(NTMAX, MINB)
    heat_window_linear_kernel(const __grid_constant__ WindowArgs a,
                              const __grid_constant__ CUtensorMap tm_r,
                              const __grid_constant__ CUtensorMap tm_fine) {
    extern __shared__ unsigned char smem_raw[];
    char* base = align1k(smem_raw);
    const int pitch = a.co.pitch;
    const int rb = row_bytes_al(pitch);
    char* bufA[2] = {base, base + rb};
    char* bufS = base + 2 * rb;
    Tabs& tb = *reinterpret_cast<Tabs*>(base + 3 * rb);
    Slots& sl = *reinterpret_cast<Slots*>(base + 3 * rb + sizeof(Tabs));
    uint64_t* barA = &sl.bar[0];  // two barriers: bar[0], bar[1]
    uint64_t* barS = &sl.bar[2];
    const uint32_t bytes = static_cast<uint32_t>(pitch * 8);
    const int R = pitch >> 4;

    Lane<L> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    tabs_init(tb, a.co);
    if (t == 0) {
        mbar_init(&barA[0], 1);
        mbar_init(&barA[1], 1);
        mbar_init(barS, 1);
        mbar_fence_init();
    }
    __syncthreads();
    uint32_t phA[2] = {0, 0}, phS = 0;

    const bool has_pre = a.pre_e1 >= a.pre_e0;
    const int n_ind = max(0, a.p1 - a.p0 + 1);
    const long long Nj = (has_pre ? 1 : 0) + n_ind;
    const int jb = static_cast<int>(Nj * blockIdx.x / gridDim.x);
    const int je = static_cast<int>(Nj * (blockIdx.x + 1) / gridDim.x);
    if (jb >= je) return;

    auto job_range = [&](int q, int& lo, int& e0, int& e1) {
        if (has_pre && q == 0) {
            lo = a.pre_lo;
            e0 = a.pre_e0;
            e1 = a.pre_e1;
        } else {
            const int p = a.p0 + q - (has_pre ? 1 : 0);
            lo = max(0, p - a.k + 1);
            e0 = e1 = p;
        }
    };
    // issue stream: (iq, is_) = next r row to load
    int iq = jb, is_, ilo, ie0, ie1;
    job_range(iq, ilo, ie0, ie1);
    is_ = ilo;
    auto issue_next = [&](int buf) {  // thread 0 only
        if (iq >= je) return;
        mbar_expect_tx(&barA[buf], bytes);
        tma_load_2d(bufA[buf], &tm_r, 0, (is_ - a.x1_base) * R, &barA[buf]);
        if (++is_ > ie1) {
            if (++iq < je) {
                job_range(iq, ilo, ie0, ie1);
                is_ = ilo;
            }
        }
    };
    if (t == 0) {
        issue_next(0);
        issue_next(1);
    }
    int cb = 0;  // buffer of the next row to consume
    double x[L];
    auto consume = [&](bool add) {
        mbar_wait(&barA[cb], phA[cb]);
        phA[cb] ^= 1;
        if (add) row_acc<L>(bufA[cb], x, ln.s, pitch, false);
        else row_load<L>(bufA[cb], x, ln.s, pitch);
        fence_proxy_async();  // generic reads before the TMA refill (WAR)
        __syncthreads();
        if (t == 0) issue_next(cb);
        cb ^= 1;
    };

    for (int q = jb; q < je; ++q) {
        int lo, e0, e1;
        job_range(q, lo, e0, e1);
        consume(false);  // e = r_lo
        if (t == 0) {
            bulk_wait_read<0>();  // S free again
            mbar_expect_tx(barS, bytes);
            tma_load_2d(bufS, &tm_fine, 0, (max(e0, lo) * a.out_stride - a.out_base) * R, barS);
        }
        for (int s = lo; s <= e1; ++s) {
            if (s > lo) {
                phi<L>(x, a.co, ln, tb, sl, s, a.forced);
                consume(true);  // e = Psi(e) + r_s
            }
            if (s >= e0) {
                // fine.u[c_s] += e
                mbar_wait(barS, phS);
                phS ^= 1;
                double y[L];
                row_load<L>(bufS, y, ln.s, pitch);
#pragma unroll
                for (int e = 0; e < L; ++e) y[e] += x[e];
                row_store<L>(bufS, y, ln.s, pitch);
                fence_proxy_async();
                __syncthreads();
                if (t == 0) {
                    tma_store_2d(&tm_fine, 0, (s * a.out_stride - a.out_base) * R, bufS);
                    bulk_commit();
                    if (s + 1 <= e1) {
                        bulk_wait_read<0>();
                        mbar_expect_tx(barS, bytes);
                        tma_load_2d(bufS, &tm_fine, 0, ((s + 1) * a.out_stride - a.out_base) * R,
                                    barS);
                    }
                }
            }
        }
    }
    if (t == 0) bulk_wait<0>();
}

// --------------------------------------------------------------------------
// generic window kernel: FAS windows (kernels.cpp:63-77), nested forward
// windows (kernels.cpp:79-88), batched single-step applications (Phi of
// given rows, forcing, Psi(v_{j-1})) and the FAS coarse right-hand side
// (solver.cpp:214-218).  smem: [O0][O1][A1][A2][A3][Tabs][Slots]

template <int L, int NTMAX, int MINB>
__global__ void __launch_bounds__(NTMAX, MINB)
    heat_window_kernel(const __grid_constant__ WindowArgs a,
                       const __grid_constant__ CUtensorMap tm_x1,
                       const __grid_constant__ CUtensorMap tm_x2,
                       const __grid_constant__ CUtensorMap tm_x3,
                       const __grid_constant__ CUtensorMap tm_out) {
    extern __shared__ unsigned char smem_raw[];
    char* base = align1k(smem_raw);
    const int pitch = a.co.pitch;
    const int rb = row_bytes_al(pitch);
    char* bufO[2] = {base, base + rb};
    char* bufA1 = base + 2 * rb;
    char* bufA2 = base + 3 * rb;
    char* bufA3 = base + 4 * rb;
    const bool three = (a.kind == WK_FAS || a.kind == WK_FAS_RHS);
    char* tl = base + (three ? 5 : 3) * rb;
    Tabs& tb = *reinterpret_cast<Tabs*>(tl);
    Slots& sl = *reinterpret_cast<Slots*>(tl + sizeof(Tabs));
    uint64_t* barA = &sl.bar[1];
    const uint32_t bytes = static_cast<uint32_t>(pitch * 8);
    const int R = pitch >> 4;

    Lane<L> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    tabs_init(tb, a.co);
    if (t == 0) {
        mbar_init(barA, 1);
        mbar_fence_init();
    }
    __syncthreads();
    uint32_t phA = 0;
    int ob = 0;

    const bool has_pre = (a.kind == WK_FAS || a.kind == WK_FORWARD) && (a.pre_e1 >= a.pre_e0);
    const int n_ind = max(0, a.p1 - a.p0 + 1);
    const long long Nj = (has_pre ? 1 : 0) + n_ind;
    const int jb = static_cast<int>(Nj * blockIdx.x / gridDim.x);
    const int je = static_cast<int>(Nj * (blockIdx.x + 1) / gridDim.x);
    double x[L];

    auto emit_store = [&](int row) {
        char* o = bufO[ob];
        row_store<L>(o, x, ln.s, pitch);
        fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            tma_store_2d(&tm_out, 0, (row - a.out_base) * R, o);
            bulk_commit();
        }
        ob ^= 1;
    };

    for (int q = jb; q < je; ++q) {
        if (a.kind == WK_APPLY || a.kind == WK_FAS_RHS) {
            const int p = a.p0 + q;
            const int src = (a.kind == WK_FAS_RHS) ? p - 1 : p + a.seed_off;
            const uint32_t nb = a.seed_zero ? 0u : bytes;
            const uint32_t extra = (a.kind == WK_FAS_RHS) ? 2 * bytes : 0u;
            if (t == 0 && nb + extra) {
                mbar_expect_tx(barA, nb + extra);
                if (!a.seed_zero) tma_load_2d(bufA1, &tm_x1, 0, (src - a.x1_base) * R, barA);
                if (a.kind == WK_FAS_RHS) {
                    tma_load_2d(bufA2, &tm_x2, 0, (p - a.x2_base) * R, barA);
                    tma_load_2d(bufA3, &tm_x3, 0, (p - a.x3_base) * R, barA);
                }
            }
            if (nb + extra) {
                mbar_wait(barA, phA);
                phA ^= 1;
            }
            if (a.seed_zero) {
#pragma unroll
                for (int e = 0; e < L; ++e) x[e] = 0.0;
            } else {
                row_load<L>(bufA1, x, ln.s, pitch);
            }
            if (t == 0) bulk_wait_read<1>();
            phi<L>(x, a.co, ln, tb, sl, a.idx0 + p, a.forced);
            if (a.kind == WK_FAS_RHS) {
                // g_j = (v_j - Psi_j(v_{j-1})) + r_j  (solver.cpp:214-218)
                double y[L];
                row_load<L>(bufA2, y, ln.s, pitch);
#pragma unroll
                for (int e = 0; e < L; ++e) y[e] -= x[e];
                row_acc<L>(bufA3, y, ln.s, pitch, false);
#pragma unroll
                for (int e = 0; e < L; ++e) x[e] = y[e];
            }
            emit_store(p);
            continue;
        }

        int lo, e0, e1;
        if (has_pre && q == 0) {
            lo = a.pre_lo;
            e0 = a.pre_e0;
            e1 = a.pre_e1;
        } else {
            const int p = a.p0 + q - (has_pre ? 1 : 0);
            lo = max(0, p - a.k + 1);
            e0 = e1 = p;
        }
        // ---- seed: v_lo + r_lo (FAS), u_lo (forward)
        const bool fas = (a.kind == WK_FAS);
        if (t == 0) {
            mbar_expect_tx(barA, fas ? 2 * bytes : bytes);
            tma_load_2d(bufA1, &tm_x1, 0, (lo - a.x1_base) * R, barA);
            if (fas) tma_load_2d(bufA2, &tm_x2, 0, (lo - a.x2_base) * R, barA);
        }
        mbar_wait(barA, phA);
        phA ^= 1;
        if (fas) {
            row_load<L>(bufA2, x, ln.s, pitch);        // v_lo
            row_acc<L>(bufA1, x, ln.s, pitch, false);  // + r_lo
        } else {
            row_load<L>(bufA1, x, ln.s, pitch);
        }
        fence_proxy_async();
        __syncthreads();
        if (lo >= e0) emit_store(lo);
        for (int s = lo + 1; s <= e1; ++s) {
            if (t == 0 && fas) {
                mbar_expect_tx(barA, 3 * bytes);
                tma_load_2d(bufA1, &tm_x1, 0, (s - a.x1_base) * R, barA);
                tma_load_2d(bufA2, &tm_x2, 0, (s - a.x2_base) * R, barA);
                tma_load_2d(bufA3, &tm_x3, 0, (s - a.x3_base) * R, barA);
            }
            if (t == 0) bulk_wait_read<1>();
            phi<L>(x, a.co, ln, tb, sl, s, a.forced);
            if (fas) {
                mbar_wait(barA, phA);
                phA ^= 1;
                // next = Psi(u) + v_s - Psi(v_{s-1}) + r_s  (kernels.cpp:69-74)
                row_acc<L>(bufA2, x, ln.s, pitch, false);
                row_acc<L>(bufA3, x, ln.s, pitch, true);
                row_acc<L>(bufA1, x, ln.s, pitch, false);
                fence_proxy_async();
                __syncthreads();
            }
            if (s >= e0) emit_store(s);
        }
    }
    if (t == 0) bulk_wait<0>();
}

// --------------------------------------------------------------------------
// host launchers

size_t heat_sweep_smem(const SweepArgs& a) {
    const int rows = 1 + a.n_out + (a.add_g ? 1 : 0);
    return 1024 + static_cast<size_t>(rows) * row_bytes_al(a.co.pitch) + sizeof(Tabs) + sizeof(Slots);
}

size_t heat_window_smem(const WindowArgs& a) {
    int rows;
    if (a.kind == WK_LINEAR) rows = 3;
    else rows = (a.kind == WK_FAS || a.kind == WK_FAS_RHS) ? 5 : 3;
    size_t pad = 0;
    if (const char* e = std::getenv("ATM_WIN_PAD")) pad = static_cast<size_t>(std::atoi(e)) * 1024;
    return pad + 1024 + static_cast<size_t>(rows) * row_bytes_al(a.co.pitch) + sizeof(Tabs) + sizeof(Slots);
}

namespace {

struct KernelPtrs {
    const void* sweep;
    const void* wlin;
    const void* win;
};

template <int L, int NT, int MB>
KernelPtrs kptrs() {
    return {reinterpret_cast<const void*>(heat_sweep_kernel<L, NT, MB>),
            reinterpret_cast<const void*>(heat_window_linear_kernel<L, NT, MB>),
            reinterpret_cast<const void*>(heat_window_kernel<L, NT, MB>)};
}

// L=16 serves 2048 < n <= 4096 with 256 threads; smaller L use up to 512
KernelPtrs select(int L) {
    switch (L) {
        case 2: return kptrs<2, 512, 1>();
        case 4: return kptrs<4, 512, 1>();
        case 8: return kptrs<8, 512, 1>();
        default: return kptrs<16, 256, 2>();
    }
}

void prepare(const void* fn) {
    static std::mutex mu;
    static std::map<const void*, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done[fn]) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    done[fn] = true;
}

int occupancy(const void* fn, int nt, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t>, int> cache;
    prepare(fn);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(fn, nt, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, nt, smem) != cudaSuccess) n = 1;
    n = std::max(1, n);
    cache[key] = n;
    return n;
}

int launch(const void* fn, int grid, int nt, size_t smem, cudaStream_t s, void** args) {
    prepare(fn);
    return static_cast<int>(cudaLaunchKernel(fn, dim3(grid), dim3(nt), args, smem, s));
}

}  // namespace

int heat_sweep_occupancy(const SweepArgs& a) {
    return occupancy(select(a.co.L).sweep, a.co.nt, heat_sweep_smem(a));
}

int heat_window_occupancy(const WindowArgs& a) {
    const KernelPtrs k = select(a.co.L);
    return occupancy(a.kind == WK_LINEAR ? k.wlin : k.win, a.co.nt, heat_window_smem(a));
}

int launch_heat_sweep(const SweepArgs& a, const CUtensorMap& u, const CUtensorMap& g,
                      const CUtensorMap& o, int grid, cudaStream_t s) {
    if (grid <= 0) return 0;
    SweepArgs aa = a;
    CUtensorMap tu = u, tg = g, to = o;
    void* args[] = {&aa, &tu, &tg, &to};
    return launch(select(a.co.L).sweep, grid, a.co.nt, heat_sweep_smem(a), s, args);
}

int launch_heat_window(const WindowArgs& a, const CUtensorMap& x1, const CUtensorMap& x2,
                       const CUtensorMap& x3, const CUtensorMap& o, int grid, cudaStream_t s) {
    if (grid <= 0) return 0;
    WindowArgs aa = a;
    CUtensorMap t1 = x1, t2 = x2, t3 = x3, to = o;
    const KernelPtrs k = select(a.co.L);
    if (a.kind == WK_LINEAR) {
        void* args[] = {&aa, &t1, &to};
        return launch(k.wlin, grid, a.co.nt, heat_window_smem(a), s, args);
    }
    void* args[] = {&aa, &t1, &t2, &t3, &to};
    return launch(k.win, grid, a.co.nt, heat_window_smem(a), s, args);
}

}  // namespace atm
