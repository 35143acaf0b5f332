// DFMA peak microbenchmark (the FP64 leg of the sweep roofline):
// every thread runs 16 independent FMA chains for `iters` rounds; the grid
// fills every SM.  Prints one JSON line: {"dfma_tflops": ..., "sm_count": ...}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 1 << 16;
    dfma_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 16.0 * iters * double(blocks) * threads;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("{\"dfma_tflops\": %.3f, \"ms\": %.3f, \"sm_count\": %d, \"max_sm_clock_mhz\": %d, "
           "\"fma_per_launch\": %.0f, \"note\": \"16 independent DFMA chains per thread, %d CTAs x %d threads, best of 5\"}\n",
           flops / (best * 1e-3) / 1e12, best, sms, clk / 1000, flops / 2, blocks, threads);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
