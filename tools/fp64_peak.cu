// FP64 peak of this B200 (roofline denominator for the on-chip kernels):
// independent DFMA chains per thread, all SMs, timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
// Prints one JSON line: DFMA/s, FP64 TFLOP/s (2 flops per DFMA), SM clock.
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 1 << 14;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 42.0) out[0] = s;  // keeps the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out = nullptr;
    cudaMalloc(&out, sizeof(double));
    const int blocks = sms * 8, threads = 256;
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(t0);
        dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, t0, t1);
        if (ms < best) best = ms;
    }
    const double dfma = static_cast<double>(blocks) * threads * kIters * kChains;
    const double rate = dfma / (best * 1e-3);
    std::printf("{\"dfma_per_s\": %.6e, \"fp64_tflops\": %.4f, \"dfma_per_clk_per_sm\": %.2f, \"sms\": %d, "
                "\"attr_clock_mhz\": %.0f, \"ms\": %.4f, \"error\": \"%s\"}\n",
                rate, 2.0 * rate / 1e12, rate / (sms * clk * 1e3), sms, clk / 1e3, best,
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
