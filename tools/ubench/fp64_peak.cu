// FP64 peak of this B200 (the secondary roofline of the Phi-chain and CG
// kernels: "measure it rather than quoting a datasheet").
// Every SM runs CTAs of independent DFMA chains (8 per thread, enough to hide
// the 8-cycle dependent-DFMA latency); CUDA events around the launch.
// Prints one JSON line: {"fp64_tflops": ..., "sm_clock_mhz": ..., ...}.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, double a, double b, int iters) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out = nullptr;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-9, 64);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-9, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * threads * blocks;
    const double tf = flops / (best * 1e-3) / 1e12;
    // per SM per clock at the attribute clock (a lower bound when boosting)
    std::printf("{\"fp64_tflops\": %.3f, \"best_ms\": %.4f, \"sms\": %d, \"clock_attr_mhz\": %.0f, "
                "\"dfma_per_sm_per_clk_at_attr\": %.3f, \"err\": \"%s\"}\n",
                tf, best, sms, clk / 1e3, flops / 2.0 / (best * 1e-3) / sms / (clk * 1e3),
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
