// HBM write-only and read-only bandwidth probes at the sweep's size (8.6 GB):
// cudaMemset, vectorised st.global, and a streaming read-sum.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void st_kernel(double2* p, size_t n2) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n2; i += stride) p[i] = make_double2(1.0, 2.0);
}
// streaming stores (st.global.cs: evict-first)
__global__ void st_cs_kernel(double2* p, size_t n2) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n2; i += stride) __stcs(p + i, make_double2(1.0, 2.0));
}
__global__ void ld_kernel(const double2* p, size_t n2, double* out) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    double s = 0;
    for (; i < n2; i += stride) { double2 v = __ldcs(p + i); s += v.x + v.y; }
    if (s == 12345.0) out[0] = s;
}
int main() {
    const size_t bytes = 8587837440ull;
    double* p; double* o;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); cudaMemsetAsync(p, 0, bytes); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("memset write: %.1f GB/s\n", bytes / ms / 1e6);
        cudaEventRecord(a); st_kernel<<<148 * 8, 512>>>((double2*)p, bytes / 16); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("st.global.v2 write: %.1f GB/s\n", bytes / ms / 1e6);
        cudaEventRecord(a); st_cs_kernel<<<148 * 8, 512>>>((double2*)p, bytes / 16); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("st.global.cs.v2 write: %.1f GB/s\n", bytes / ms / 1e6);
        cudaEventRecord(a); ld_kernel<<<148 * 8, 512>>>((const double2*)p, bytes / 16, o); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("ld read: %.1f GB/s\n", bytes / ms / 1e6);
        cudaEventRecord(a); cudaMemcpyAsync(p + bytes / 16, p, bytes / 2, cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); printf("d2d copy (r+w): %.1f GB/s\n", bytes / ms / 1e6);
    }
    return 0;
}
