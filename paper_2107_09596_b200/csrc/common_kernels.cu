// common_kernels.cu -- seeded fills, row arithmetic, deterministic norm
// reduction, and the scalar (n = 1) Phi backend.
#include <algorithm>
#include <climits>
#include <cmath>

#include "common_kernels.cuh"
#include "heat_kernels.cuh"

namespace atm {

// ---------------------------------------------------------------------------
// seeded fill (state_vector.hpp:92-118).  Draw q of point i is
// mix(seed_i + (q+1)*golden) -- integer arithmetic, exact conversion, so the
// device fill is bitwise equal to the reference's sequential generator.

__device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void fill_random_kernel(double* u, int row0, int pitch, int n, int i0, int rows,
                                   int step, uint64_t seed) {
    const long long total = static_cast<long long>(rows) * n;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx / n);
        const int i = i0 + r * step;
        const int q = static_cast<int>(idx % n);
        const uint64_t st = (seed + static_cast<uint64_t>(i)) +
                            static_cast<uint64_t>(q + 1) * 0x9E3779B97F4A7C15ULL;
        const double unit = static_cast<double>(sm64_mix(st) >> 11) * 0x1.0p-53;
        u[static_cast<size_t>(row0 + r) * pitch + q] = 2.0 * unit - 1.0;
    }
}

// rows i = i0, i0 + step, ... < i1 (step > 1: C-point-only arrays, row (i - base) / step)
int launch_fill_random(double* u, int base, int pitch, int n, int i0, int i1, uint64_t seed,
                       cudaStream_t s, int step) {
    if (i1 <= i0) return 0;
    const int rows = (i1 - i0 + step - 1) / step;
    const long long total = static_cast<long long>(rows) * n;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
    fill_random_kernel<<<blocks, 256, 0, s>>>(u, (i0 - base) / step, pitch, n, i0, rows, step, seed);
    return static_cast<int>(cudaGetLastError());
}

__global__ void fill_rows_kernel(double* u, int base, int pitch, int n, int i0, int i1,
                                 const double* v) {
    const long long total = static_cast<long long>(i1 - i0) * n;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = i0 + static_cast<int>(idx / n);
        const int q = static_cast<int>(idx % n);
        u[static_cast<size_t>(i - base) * pitch + q] = v[q];
    }
}

int launch_fill_rows(double* u, int base, int pitch, int n, int i0, int i1, const double* v,
                     cudaStream_t s) {
    if (i1 <= i0) return 0;
    const long long total = static_cast<long long>(i1 - i0) * n;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
    fill_rows_kernel<<<blocks, 256, 0, s>>>(u, base, pitch, n, i0, i1, v);
    return static_cast<int>(cudaGetLastError());
}

// r = g - u over one row (residual at point 0, kernels.cpp:35-37)
__global__ void row_diff_kernel(double* r, const double* g, const double* u, int n, double* sq) {
    __shared__ double red[32];
    double s = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const double d = g[q] - u[q];
        r[q] = d;
        s = fma(d, d, s);
    }
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0 && sq) {
        double tot = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
        sq[0] = tot;
    }
}

int launch_row_diff(double* r, const double* g, const double* u, int n, double* sq,
                    cudaStream_t s) {
    row_diff_kernel<<<1, 256, 0, s>>>(r, g, u, n, sq);
    return static_cast<int>(cudaGetLastError());
}

__global__ void c_correct_kernel(double* u, int u_base, int m, const double* cu,
                                 const double* cv, int c_base, int pitch, int n, int j0, int j1) {
    const long long total = static_cast<long long>(j1 - j0) * n;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         idx < total; idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = j0 + static_cast<int>(idx / n);
        const int q = static_cast<int>(idx % n);
        const size_t cr = static_cast<size_t>(j - c_base) * pitch + q;
        const double e = cu[cr] - cv[cr];
        u[static_cast<size_t>(j * m - u_base) * pitch + q] += e;
    }
}

int launch_c_correct(double* u, int u_base, int m, const double* cu, const double* cv,
                     int c_base, int pitch, int n, int j0, int j1, cudaStream_t s) {
    if (j1 <= j0) return 0;
    const long long total = static_cast<long long>(j1 - j0) * n;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
    c_correct_kernel<<<blocks, 256, 0, s>>>(u, u_base, m, cu, cv, c_base, pitch, n, j0, j1);
    return static_cast<int>(cudaGetLastError());
}

__global__ void row_sum_kernel(double* g, const double* v, const double* r, int n) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        g[q] = v[q] + r[q];
}

int launch_row_sum(double* g, const double* v, const double* r, int n, cudaStream_t s) {
    row_sum_kernel<<<(n + 255) / 256, 256, 0, s>>>(g, v, r, n);
    return static_cast<int>(cudaGetLastError());
}

// Fixed association in two stages: block b sums slice b of 256 equal slices
// (thread t takes elements t, t+256, ... of the slice in order, then a fixed
// binary tree), the last block to finish sums the 256 partials the same way.
// Depends only on `count`, so every shard decomposition yields the same bits
// (the reference sums in point order for the same reason, parallel.cpp:279-295).
constexpr int kNormBlocks = 256;

__device__ double block_tree_sum(double s, double* part) {
    const int t = threadIdx.x;
    part[t] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
        if (t < w) part[t] = part[t] + part[t + w];
        __syncthreads();
    }
    return part[0];
}

__global__ void norm_kernel(const double* sq, int count, double* partials, unsigned* ticket,
                            double* out) {
    __shared__ double part[256];
    __shared__ bool last;
    const long long lo = static_cast<long long>(count) * blockIdx.x / kNormBlocks;
    const long long hi = static_cast<long long>(count) * (blockIdx.x + 1) / kNormBlocks;
    double s = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) s += sq[i];
    const double tot = block_tree_sum(s, part);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = tot;
        __threadfence();
        last = (atomicAdd(ticket, 1u) == kNormBlocks - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const double v = reinterpret_cast<volatile double*>(partials)[threadIdx.x];
    const double all = block_tree_sum(v, part);
    if (threadIdx.x == 0) {
        out[0] = sqrt(all);
        *ticket = 0;  // ready for the next launch (stream-ordered)
    }
}

int launch_norm_from_squares(const double* sq, int count, double* out, cudaStream_t s) {
    // out[0] = norm; out[8..8+256) partials; the ticket lives at out[4]
    norm_kernel<<<kNormBlocks, 256, 0, s>>>(sq, count, out + 8, reinterpret_cast<unsigned*>(out + 4),
                                           out);
    return static_cast<int>(cudaGetLastError());
}

__global__ void functional_kernel(const double* u, int u_base, int m, int pitch, int n,
                                  const double* w, double* prev, int j0, int j1,
                                  unsigned long long* out_max, int init) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int j = j0 + blockIdx.x * wpb + (threadIdx.x >> 5); j < j1; j += gridDim.x * wpb) {
        const double* row = u + static_cast<size_t>(j * m - u_base) * pitch;
        // lane-strided partial sums in index order, then a fixed xor tree:
        // deterministic, the same for any grid or shard count
        double s = 0.0;
        if (w) {
            for (int q = lane; q < n; q += 32) s = __dadd_rn(s, __dmul_rn(w[q], row[q]));
        } else {
            for (int q = lane; q < n; q += 32) s = __dadd_rn(s, __dmul_rn(row[q], row[q]));
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
        const double val = w ? s : sqrt(s);
        if (lane == 0) {
            if (!init) {
                const double p = prev[j];
                const double rel = fabs(val - p) / fmax(fabs(p), 1e-300);
                // rel >= 0: the bit pattern orders like the value (+inf last)
                if (rel > 0.0) atomicMax(out_max, static_cast<unsigned long long>(__double_as_longlong(rel)));
            }
            prev[j] = val;
        }
    }
}

int launch_functional(const double* u, int u_base, int m, int pitch, int n, const double* w,
                      double* prev, int j0, int j1, double* out_max, int init, cudaStream_t s) {
    if (j1 <= j0) return 0;
    if (!init) {
        const cudaError_t e = cudaMemsetAsync(out_max, 0, sizeof(double), s);
        if (e != cudaSuccess) return static_cast<int>(e);
    }
    const int warps = 8, blocks = std::min((j1 - j0 + warps - 1) / warps, 148 * 8);
    functional_kernel<<<blocks, warps * 32, 0, s>>>(u, u_base, m, pitch, n, w, prev, j0, j1,
                                                   reinterpret_cast<unsigned long long*>(out_max), init);
    return static_cast<int>(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// scalar backend: one thread per job, same job semantics as the heat kernels

__device__ __forceinline__ double sc_phi(const ScalarCoefDev& co, int index, double u) {
    double v = co.mult * u;
    if (co.ff) v += co.ff[index];
    return v;
}

__global__ void scalar_sweep_kernel(ScalarSweepArgs a) {
    const int J = a.j0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (J >= a.j1) return;
    const int m = a.m, last = a.np - 1, c = J * m;
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
    const int ud = a.u_div > 1 ? a.u_div : 1;
    double x = a.u[(start - a.u_base) / ud];
    for (int i = start + 1; i <= end; ++i) {
        x = sc_phi(a.co, i, x);
        if (a.add_g) x += a.g[i - a.g_base];
        if (i >= store_from && store_row(a.store, i, m)) a.u[i - a.u_base] = x;
    }
    if (a.tail != TAIL_NONE && end + 1 <= last && ((end + 1) % m) == 0) {
        const int ti = end + 1;
        double r = sc_phi(a.co, ti, x);
        if (a.add_g) r += a.g[ti - a.g_base];
        r -= a.u[(ti - a.u_base) / ud];
        const int ci = ti / m;
        if (a.tail == TAIL_STORE || a.tail == TAIL_BOTH) a.out[ci - a.out_base] = r;
        if (a.tail == TAIL_SQ || a.tail == TAIL_BOTH) a.sq[(ti - a.sq_base) / a.sq_div] = r * r;
    }
}

int launch_scalar_sweep(const ScalarSweepArgs& a, cudaStream_t s) {
    const int n = a.j1 - a.j0;
    if (n <= 0) return 0;
    scalar_sweep_kernel<<<(n + 127) / 128, 128, 0, s>>>(a);
    return static_cast<int>(cudaGetLastError());
}

__global__ void scalar_window_kernel(ScalarWindowArgs a) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (a.kind == WK_APPLY || a.kind == WK_FAS_RHS) {
        const int p = a.p0 + q;
        if (p > a.p1) return;
        if (a.kind == WK_APPLY) {
            const double x0 = a.seed_zero ? 0.0 : a.x1[p + a.seed_off - a.x1_base];
            a.out[p - a.out_base] = sc_phi(a.co, a.idx0 + p, x0);
        } else {
            const double psi = sc_phi(a.co, p, a.x1[p - 1 - a.x1_base]);
            double y = a.x2[p - a.x2_base];
            y -= psi;
            y += a.x3[p - a.x3_base];
            a.out[p - a.out_base] = y;
        }
        return;
    }
    const bool has_pre = a.pre_e1 >= a.pre_e0;
    const int nj = (has_pre ? 1 : 0) + max(0, a.p1 - a.p0 + 1);
    if (q >= nj) return;
    int lo, e0, e1;
    if (has_pre && q == 0) {
        lo = a.pre_lo; e0 = a.pre_e0; e1 = a.pre_e1;
    } else {
        const int p = a.p0 + q - (has_pre ? 1 : 0);
        lo = max(0, p - a.k + 1);
        e0 = e1 = p;
    }
    double x;
    if (a.kind == WK_FAS) x = a.x2[lo - a.x2_base] + a.x1[lo - a.x1_base];
    else x = a.x1[lo - a.x1_base];
    auto emit = [&](int p) {
        if (a.kind == WK_LINEAR) a.out[p * a.out_stride - a.out_base] += x;
        else a.out[p - a.out_base] = x;
    };
    if (lo >= e0) emit(lo);
    for (int s = lo + 1; s <= e1; ++s) {
        double y = sc_phi(a.co, s, x);
        if (a.kind == WK_LINEAR) {
            y += a.x1[s - a.x1_base];
        } else if (a.kind == WK_FAS) {
            y += a.x2[s - a.x2_base];
            y -= a.x3[s - a.x3_base];
            y += a.x1[s - a.x1_base];
        }
        x = y;
        if (s >= e0) emit(s);
    }
}

int launch_scalar_window(const ScalarWindowArgs& a, cudaStream_t s) {
    int nj;
    if (a.kind == WK_APPLY || a.kind == WK_FAS_RHS) nj = a.p1 - a.p0 + 1;
    else nj = ((a.pre_e1 >= a.pre_e0) ? 1 : 0) + std::max(0, a.p1 - a.p0 + 1);
    if (nj <= 0) return 0;
    scalar_window_kernel<<<(nj + 127) / 128, 128, 0, s>>>(a);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace atm
