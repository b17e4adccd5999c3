// heat_kernels.cu -- Heat1D Phi chains for sm_100a.
//
// One CTA owns one state vector (a time point) in registers, blocked
// (thread t holds elements [t*L, t*L+L)).  Rows move HBM <-> smem by TMA
// (cp.async.bulk.tensor, 128B-swizzled so the blocked register view reads
// and writes smem conflict-free); produced rows leave through a double-
// buffered TMA-store staging area so stores overlap the next Phi.
//
// Reference semantics restated (file:line under /root/reference/proj):
//   Phi / step          heat1d.cpp:47-60 (Thomas), :66-83 (sub-steps, forcing)
//   F-relaxation        kernels.cpp:7-17      -> SW_F jobs
//   C-relaxation        kernels.cpp:19-28     -> SW_CRELAX jobs / fused SW_FCF
//   residual / restrict kernels.cpp:30-43, solver.cpp:174-185 -> tails, SW_RESID
//   window solves       kernels.cpp:53-88     -> heat_window_kernel
//   point squares       kernels.cpp:90-95     -> TAIL_SQ (fixed-order tree)
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>

#include "heat_kernels.cuh"
#include "tma.cuh"

namespace atm {

// --------------------------------------------------------------------------
// host: coefficients and scan multipliers

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
    // coefficients agree with their limit to <= 2 ulp and are held in registers
    H.i0 = n;
    if (n >= 3) {
        const double bc = beta[n - 2], cc = -cpr[n - 2];
        auto close = [](double x, double y) {
            return std::fabs(x - y) <= 4.5e-16 * std::fabs(y);
        };
        int last_diff = -1;
        for (int i = 0; i < n - 1; ++i)
            if (!close(beta[i], bc) || !close(-cpr[i], cc)) last_diff = i;
        H.i0 = ((last_diff + 1 + L - 1) / L) * L;
        H.beta_c = bc;
        H.gamma_c = H.r * bc;
        H.cneg_c = cc;
    }
    // effective per-element coefficients as the device will use them
    std::vector<double> eg(npad), ec(npad);
    for (int t = 0; t < nt; ++t) {
        const int s = t * L;
        const bool cst = (s >= H.i0) && (s + L <= n - 1);
        for (int e = 0; e < L; ++e) {
            eg[s + e] = cst ? H.gamma_c : H.gamma[s + e];
            ec[s + e] = cst ? H.cneg_c : H.cneg[s + e];
        }
    }
    std::vector<double> Af(nt, 1.0), Ab(nt, 1.0);
    for (int t = 0; t < nt; ++t) {
        for (int e = 0; e < L; ++e) Af[t] *= eg[t * L + e];
        for (int e = L - 1; e >= 0; --e) Ab[t] *= ec[t * L + e];
    }
    H.scan.assign(static_cast<size_t>(nt) * kScanPerThread, 0.0);
    H.warpA.assign(2 * kMaxWarps, 0.0);
    const int nw = nt / 32;
    for (int w = 0; w < nw; ++w) {
        double pf = 1.0, pb = 1.0;
        for (int l = 0; l < 32; ++l) pf *= Af[32 * w + l];
        for (int l = 31; l >= 0; --l) pb *= Ab[32 * w + l];
        H.warpA[w] = pf;
        H.warpA[kMaxWarps + w] = pb;
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
    return H;
}

// --------------------------------------------------------------------------
// device: per-thread state and the tridiagonal solve

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

struct Slots {            // small shared scratch
    double swf[kMaxWarps];
    double swb[kMaxWarps];
    double wAf[kMaxWarps];
    double wAb[kMaxWarps];
    double red[kMaxWarps];
    uint64_t bar[4];
};

// (I + sub_dt L) x = x, in place, over the CTA (heat1d.cpp:47-60).
template <int L>
__device__ __forceinline__ void tri_solve(double (&x)[L], const HeatCoefDev& co,
                                          const Lane<L>& ln, Slots& sl) {
    const double r = co.r;
    // forward: y_i = (x_i + r y_{i-1}) / den_i, local with zero carry-in
    double y = 0.0;
    if (ln.cst) {
        const double b = co.beta_c;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            y = fma(r, y, x[e]) * b;
            x[e] = y;
        }
    } else {
        const double* bt = co.beta + ln.s;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            y = fma(r, y, x[e]) * __ldg(bt + e);
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
    double cw = 0.0;
    for (int v = 0; v < ln.warp; ++v) cw = fma(sl.wAf[v], cw, sl.swf[v]);
    double p = fma(ln.Pfex, cw, ex);
    if (ln.cst) {
        const double g = co.gamma_c;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            p *= g;
            x[e] += p;
        }
    } else {
        const double* gt = co.gamma + ln.s;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            p *= __ldg(gt + e);
            x[e] += p;
        }
    }
    // backward: x_i = y_i - c'_i x_{i+1}, local with zero carry-in
    double z = 0.0;
    if (ln.cst) {
        const double c = co.cneg_c;
#pragma unroll
        for (int e = L - 1; e >= 0; --e) {
            z = fma(c, z, x[e]);
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
    cw = 0.0;
    for (int v = ln.nw - 1; v > ln.warp; --v) cw = fma(sl.wAb[v], cw, sl.swb[v]);
    p = fma(ln.Pbex, cw, ex);
    if (ln.cst) {
        const double c = co.cneg_c;
#pragma unroll
        for (int e = L - 1; e >= 0; --e) {
            p *= c;
            x[e] += p;
        }
    } else {
        const double* ct = co.cneg + ln.s;
#pragma unroll
        for (int e = L - 1; e >= 0; --e) {
            p *= __ldg(ct + e);
            x[e] += p;
        }
    }
}

// Phi_index on this level: S sub-steps, forcing added before each solve
// when `forced` (heat1d.cpp:66-83).
template <int L>
__device__ __forceinline__ void phi(double (&x)[L], const HeatCoefDev& co, const Lane<L>& ln,
                                    Slots& sl, int index, int forced) {
    for (int s = 0; s < co.substeps; ++s) {
        if (forced) {
            const double th = __ldg(co.theta + static_cast<size_t>(index) * co.substeps + s);
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(th, __ldg(co.prof + ln.s + e), x[e]);
        }
        tri_solve<L>(x, co, ln, sl);
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

// x = x + row  (sign = +1) or x = x - row (sign = -1)
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

// y = row + x (row first operand, matches u.add(e) ordering is commutative anyway)
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

template <int L>
__global__ void __launch_bounds__(kMaxThreads)
    heat_sweep_kernel(const __grid_constant__ SweepArgs a, const __grid_constant__ CUtensorMap tm_u,
                      const __grid_constant__ CUtensorMap tm_g,
                      const __grid_constant__ CUtensorMap tm_out) {
    extern __shared__ unsigned char smem_raw[];
    char* base = align1k(smem_raw);
    const int pitch = a.co.pitch;
    const int rb = row_bytes_al(pitch);
    char* bufO[2] = {base, base + rb};
    char* bufS = base + 2 * rb;
    char* bufA = base + 3 * rb;
    Slots& sl = *reinterpret_cast<Slots*>(base + (a.add_g ? 4 : 3) * rb);
    uint64_t* barS = &sl.bar[0];
    uint64_t* barA = &sl.bar[1];
    const uint32_t bytes = static_cast<uint32_t>(pitch * 8);
    const int R = pitch >> 4;

    Lane<L> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    if (t < ln.nw) {
        sl.wAf[t] = a.co.warpA[t];
        sl.wAb[t] = a.co.warpA[kMaxWarps + t];
    }
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
            if (t == 0) bulk_wait_read<1>();
            phi<L>(x, a.co, ln, sl, i, a.forced);
            if (a.add_g) {
                mbar_wait(barA, phA);
                phA ^= 1;
                row_acc<L>(bufA, x, ln.s, pitch, false);
            }
            if (a.store && i >= store_from) {
                char* o = bufO[ob];
                row_store<L>(o, x, ln.s, pitch);
                fence_proxy_async();
                __syncthreads();
                if (t == 0) {
                    tma_store_2d(&tm_u, 0, (i - a.u_base) * R, o);
                    bulk_commit();
                }
                ob ^= 1;
            } else if (a.add_g) {
                __syncthreads();  // bufA consumed before the next load
            }
        }

        // ---- tail: residual at the next C-point, r = Phi(u_last) + g_c - u_c
        if (tail_i >= 0) {
            if (a.add_g && t == 0) {
                mbar_expect_tx(barA, bytes);
                tma_load_2d(bufA, &tm_g, 0, (tail_i - a.g_base) * R, barA);
            }
            if (t == 0) bulk_wait_read<1>();
            phi<L>(x, a.co, ln, sl, tail_i, a.forced);
            if (a.add_g) {
                mbar_wait(barA, phA);
                phA ^= 1;
                row_acc<L>(bufA, x, ln.s, pitch, false);
            }
            mbar_wait(barS, phS);
            phS ^= 1;
            row_acc<L>(bufS, x, ln.s, pitch, true);
            if (a.kind == SW_F && J + 1 < je) seed_ready = true;  // S holds u[c_{J+1}]
            const int ci = tail_i / m;
            if (a.tail == TAIL_STORE) {
                char* o = bufO[ob];
                row_store<L>(o, x, ln.s, pitch);
                fence_proxy_async();
                __syncthreads();
                if (t == 0) {
                    tma_store_2d(&tm_out, 0, (ci - a.out_base) * R, o);
                    bulk_commit();
                }
                ob ^= 1;
            } else {
                const double tot = cta_sum_squares<L>(x, ln, sl);
                if (t == 0) a.sq[tail_i - a.sq_base] = tot;
            }
        }
    }
    if (t == 0) bulk_wait<0>();
}

// --------------------------------------------------------------------------
// window kernel: truncated local coarse grids (kernels.cpp:53-88) and
// batched single-step applications

template <int L>
__global__ void __launch_bounds__(kMaxThreads)
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
    char* bufS = base + 2 * rb;
    char* bufA1 = base + 3 * rb;
    char* bufA2 = base + 4 * rb;
    char* bufA3 = base + 5 * rb;
    const bool three = (a.kind == WK_FAS || a.kind == WK_FAS_RHS);
    Slots& sl = *reinterpret_cast<Slots*>(base + (three ? 6 : 4) * rb);
    uint64_t* barS = &sl.bar[0];
    uint64_t* barA = &sl.bar[1];
    const uint32_t bytes = static_cast<uint32_t>(pitch * 8);
    const int R = pitch >> 4;

    Lane<L> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    if (t < ln.nw) {
        sl.wAf[t] = a.co.warpA[t];
        sl.wAb[t] = a.co.warpA[kMaxWarps + t];
    }
    if (t == 0) {
        mbar_init(barS, 1);
        mbar_init(barA, 1);
        mbar_fence_init();
    }
    __syncthreads();
    uint32_t phS = 0, phA = 0;
    int ob = 0;

    const bool has_pre = (a.kind <= WK_FORWARD) && (a.pre_e1 >= a.pre_e0);
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
            if (t == 0) {
                const uint32_t nb = a.seed_zero ? 0u : bytes;
                const uint32_t extra = (a.kind == WK_FAS_RHS) ? 2 * bytes : 0u;
                if (nb + extra) mbar_expect_tx(barA, nb + extra);
                if (!a.seed_zero) tma_load_2d(bufA1, &tm_x1, 0, (src - a.x1_base) * R, barA);
                if (a.kind == WK_FAS_RHS) {
                    tma_load_2d(bufA2, &tm_x2, 0, (p - a.x2_base) * R, barA);
                    tma_load_2d(bufA3, &tm_x3, 0, (p - a.x3_base) * R, barA);
                }
            }
            const bool waited = !(a.seed_zero && a.kind == WK_APPLY);
            if (waited) {
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
            phi<L>(x, a.co, ln, sl, a.idx0 + p, a.forced);
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
        // ---- seed: r_lo (linear), v_lo + r_lo (FAS), u_lo (forward)
        if (t == 0) {
            const bool fas = (a.kind == WK_FAS);
            mbar_expect_tx(barA, fas ? 2 * bytes : bytes);
            tma_load_2d(bufA1, &tm_x1, 0, (lo - a.x1_base) * R, barA);
            if (fas) tma_load_2d(bufA2, &tm_x2, 0, (lo - a.x2_base) * R, barA);
        }
        mbar_wait(barA, phA);
        phA ^= 1;
        if (a.kind == WK_FAS) {
            row_load<L>(bufA2, x, ln.s, pitch);   // v_lo
            row_acc<L>(bufA1, x, ln.s, pitch, false);  // + r_lo
        } else {
            row_load<L>(bufA1, x, ln.s, pitch);
        }
        __syncthreads();
        int next_emit = max(e0, lo);
        if (a.kind == WK_LINEAR && t == 0) {
            mbar_expect_tx(barS, bytes);
            tma_load_2d(bufS, &tm_out, 0, (next_emit * a.out_stride - a.out_base) * R, barS);
        }
        auto emit = [&](int p) {
            if (a.kind == WK_LINEAR) {
                // fine.u[c_p] += e  (solver.cpp:277)
                mbar_wait(barS, phS);
                phS ^= 1;
                double y[L];
                row_load<L>(bufS, y, ln.s, pitch);
#pragma unroll
                for (int e = 0; e < L; ++e) y[e] += x[e];
                char* o = bufO[ob];
                row_store<L>(o, y, ln.s, pitch);
                fence_proxy_async();
                __syncthreads();
                if (t == 0) {
                    tma_store_2d(&tm_out, 0, (p * a.out_stride - a.out_base) * R, o);
                    bulk_commit();
                    if (p + 1 <= e1) {
                        mbar_expect_tx(barS, bytes);
                        tma_load_2d(bufS, &tm_out, 0, ((p + 1) * a.out_stride - a.out_base) * R,
                                    barS);
                    }
                }
                ob ^= 1;
            } else {
                emit_store(p);
            }
        };
        if (lo >= e0) emit(lo);
        for (int s = lo + 1; s <= e1; ++s) {
            if (t == 0 && a.kind != WK_FORWARD) {
                const bool fas = (a.kind == WK_FAS);
                mbar_expect_tx(barA, fas ? 3 * bytes : bytes);
                tma_load_2d(bufA1, &tm_x1, 0, (s - a.x1_base) * R, barA);
                if (fas) {
                    tma_load_2d(bufA2, &tm_x2, 0, (s - a.x2_base) * R, barA);
                    tma_load_2d(bufA3, &tm_x3, 0, (s - a.x3_base) * R, barA);
                }
            }
            if (t == 0) bulk_wait_read<1>();
            phi<L>(x, a.co, ln, sl, s, a.forced);
            if (a.kind != WK_FORWARD) {
                mbar_wait(barA, phA);
                phA ^= 1;
                if (a.kind == WK_FAS) {
                    // next = Psi(u) + v_s - Psi(v_{s-1}) + r_s  (kernels.cpp:69-74)
                    row_acc<L>(bufA2, x, ln.s, pitch, false);
                    row_acc<L>(bufA3, x, ln.s, pitch, true);
                    row_acc<L>(bufA1, x, ln.s, pitch, false);
                } else {
                    row_acc<L>(bufA1, x, ln.s, pitch, false);  // e = Psi(e) + r_s
                }
                __syncthreads();
            }
            if (s >= e0) emit(s);
        }
    }
    if (t == 0) bulk_wait<0>();
}

// --------------------------------------------------------------------------
// host launchers

size_t heat_sweep_smem(const SweepArgs& a) {
    return 1024 + static_cast<size_t>(a.add_g ? 4 : 3) * row_bytes_al(a.co.pitch) + sizeof(Slots);
}

size_t heat_window_smem(const WindowArgs& a) {
    const bool three = (a.kind == WK_FAS || a.kind == WK_FAS_RHS);
    return 1024 + static_cast<size_t>(three ? 6 : 4) * row_bytes_al(a.co.pitch) + sizeof(Slots);
}

template <int L>
static int launch_sweep_L(const SweepArgs& a, const CUtensorMap& u, const CUtensorMap& g,
                          const CUtensorMap& o, int grid, cudaStream_t s) {
    const size_t smem = heat_sweep_smem(a);
    cudaFuncSetAttribute(heat_sweep_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    heat_sweep_kernel<L><<<grid, a.co.nt, smem, s>>>(a, u, g, o);
    return static_cast<int>(cudaGetLastError());
}

template <int L>
static int launch_window_L(const WindowArgs& a, const CUtensorMap& x1, const CUtensorMap& x2,
                           const CUtensorMap& x3, const CUtensorMap& o, int grid, cudaStream_t s) {
    const size_t smem = heat_window_smem(a);
    cudaFuncSetAttribute(heat_window_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    heat_window_kernel<L><<<grid, a.co.nt, smem, s>>>(a, x1, x2, x3, o);
    return static_cast<int>(cudaGetLastError());
}

int launch_heat_sweep(const SweepArgs& a, const CUtensorMap& u, const CUtensorMap& g,
                      const CUtensorMap& o, int grid, cudaStream_t s) {
    switch (a.co.L) {
        case 2: return launch_sweep_L<2>(a, u, g, o, grid, s);
        case 4: return launch_sweep_L<4>(a, u, g, o, grid, s);
        case 8: return launch_sweep_L<8>(a, u, g, o, grid, s);
        case 16: return launch_sweep_L<16>(a, u, g, o, grid, s);
    }
    return static_cast<int>(cudaErrorInvalidValue);
}

int launch_heat_window(const WindowArgs& a, const CUtensorMap& x1, const CUtensorMap& x2,
                       const CUtensorMap& x3, const CUtensorMap& o, int grid, cudaStream_t s) {
    switch (a.co.L) {
        case 2: return launch_window_L<2>(a, x1, x2, x3, o, grid, s);
        case 4: return launch_window_L<4>(a, x1, x2, x3, o, grid, s);
        case 8: return launch_window_L<8>(a, x1, x2, x3, o, grid, s);
        case 16: return launch_window_L<16>(a, x1, x2, x3, o, grid, s);
    }
    return static_cast<int>(cudaErrorInvalidValue);
}

int heat_max_ctas_per_sm(int L, int nt, size_t smem, bool window) {
    int n = 0;
    const void* fn = nullptr;
    switch (L) {
        case 2: fn = window ? (const void*)heat_window_kernel<2> : (const void*)heat_sweep_kernel<2>; break;
        case 4: fn = window ? (const void*)heat_window_kernel<4> : (const void*)heat_sweep_kernel<4>; break;
        case 8: fn = window ? (const void*)heat_window_kernel<8> : (const void*)heat_sweep_kernel<8>; break;
        case 16: fn = window ? (const void*)heat_window_kernel<16> : (const void*)heat_sweep_kernel<16>; break;
        default: return 1;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, nt, smem) != cudaSuccess) return 1;
    return std::max(1, n);
}

}  // namespace atm
