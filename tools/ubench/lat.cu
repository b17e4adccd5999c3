// latency / throughput probes for the Phi inner ops (DFMA chain, 64-bit SHFL,
// LDS, BAR) on one SM; prints cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* cyc, double a, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fma(a, x, 1.0);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, double a, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = __shfl_up_sync(0xffffffffu, x, 1) + a;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl_fma(double* out, long long* cyc, double a, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fma(a, __shfl_up_sync(0xffffffffu, x, 1), x);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, long long* cyc, double a, int n) {
    __shared__ double s[1024];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s[threadIdx.x] = x;
        __syncthreads();
        x = s[(threadIdx.x + 32) & (blockDim.x - 1)] * a;
        __syncthreads();
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: independent DFMA streams per thread
__global__ void k_dfma_tp(double* out, long long* cyc, double a, int n) {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(a, x[j], 1.0);
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < 8; ++j) s += x[j];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// single-warp issue rate: NI independent DFMA chains per thread
template <int NI>
__global__ void k_dfma_ilp(double* out, long long* cyc, double a, int n) {
    double x[NI];
    for (int j = 0; j < NI; ++j) x[j] = threadIdx.x + j;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < NI; ++j) x[j] = fma(a, x[j], 1.0);
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < NI; ++j) s += x[j];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NI>
void run_ilp(double* o, long long* c, int n) {
    long long h;
    for (int nt : {32, 64, 128, 256, 384}) {
        k_dfma_ilp<NI><<<1, nt>>>(o, c, 0.999, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA ILP %d, %d thr: %.2f cyc per warp-DFMA per warp, %.3f warp-DFMA/cyc/SM\n", NI, nt,
               double(h) / (double(NI) * n), (nt / 32) * double(NI) * n / double(h));
    }
}
int main() {
    double* o; long long* c; long long h;
    cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
    const int n = 1000;
    k_dfma<<<1, 32>>>(o, c, 0.999, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dep latency: %.2f cyc\n", double(h) / (16.0 * n));
    k_shfl<<<1, 32>>>(o, c, 0.5, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("SHFL64+DADD dep: %.2f cyc\n", double(h) / (16.0 * n));
    k_shfl_fma<<<1, 32>>>(o, c, 0.5, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("SHFL64+DFMA scan step: %.2f cyc\n", double(h) / (16.0 * n));
    for (int nt : {32, 256, 512}) {
        k_bar<<<1, nt>>>(o, c, 0.5, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("STS+BAR+LDS+BAR (%d thr): %.2f cyc\n", nt, double(h) / n);
    }
    for (int nt : {32, 128, 256, 512, 1024}) {
        k_dfma_tp<<<1, nt>>>(o, c, 0.999, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput %d thr: %.3f warp-DFMA/cyc/SM\n", nt, (nt / 32) * 8.0 * n / double(h));
    }
    run_ilp<1>(o, c, n);
    run_ilp<2>(o, c, n);
    run_ilp<4>(o, c, n);
    run_ilp<8>(o, c, n);
    run_ilp<16>(o, c, n);
    return 0;
}
