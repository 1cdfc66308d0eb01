// Does a warp shuffle compete with shared-memory loads for the same data
// pipe?  Three loops per thread -- 64-bit shared loads (conflict-free),
// 64-bit shuffles (two SHFL.32), and both interleaved -- timed alone on all
// SMs (512 threads per CTA, one CTA per SM).  If "both" takes the sum of the
// two, shuffles are no way around a shared-memory-bound stencil; if it takes
// the larger of the two, neighbour exchange by shuffle is free next to LDS.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o shfl_bench tools/shfl_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(double* out, int iters) {
    __shared__ double buf[2048];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2048; i += 512) buf[i] = 1.0 + i * 1e-6;
    __syncthreads();
    // independent chains: four shared-load sums and four shuffled values
    double a[4] = {tid * 1e-3, 0.5, 0.25, 0.125};
    double b[4] = {1.0 + tid, 2.0 + tid, 3.0 + tid, 4.0 + tid};
    int idx = tid;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (MODE & 1) {
                a[u] += buf[(idx + 67 * u) & 2047];
                a[u] += buf[(idx + 67 * u + 512) & 2047];
            }
            if (MODE & 2) {
                b[u] = __shfl_down_sync(0xffffffffu, b[u], 1);
                b[u] = __shfl_up_sync(0xffffffffu, b[u], 1) + 1.0;
            }
        }
        idx = (idx + 1) & 2047;
    }
    const double a0 = a[0] + a[1] + b[0] + b[1], a1 = a[2] + b[2], a2 = a[3], a3 = b[3];
    out[blockIdx.x * 512 + tid] = a0 + a1 + a2 + a3;
}

template <int MODE>
float run(double* d, int iters, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<MODE><<<sms, 512>>>(d, iters);
    cudaEventRecord(e0);
    bench<MODE><<<sms, 512>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, sizeof(double) * 512 * sms);
    const int iters = 20000;
    const float lds = run<1>(d, iters, sms), shf = run<2>(d, iters, sms), both = run<3>(d, iters, sms);
    // per iteration and warp: 8 LDS.64 (16 wavefronts), 8 64-bit shuffles (16 SHFL.32)
    const double clk = 1.965e6;  // cycles per ms
    printf("{\"sms\": %d, \"lds_ms\": %.3f, \"shfl_ms\": %.3f, \"both_ms\": %.3f, "
           "\"lds_cycles_per_warp_ld64\": %.2f, \"shfl_cycles_per_warp_shfl64\": %.2f, \"both_over_sum\": %.3f, "
           "\"both_over_max\": %.3f}\n",
           sms, lds, shf, both, lds * clk / (iters * 8.0 * 16), shf * clk / (iters * 8.0 * 16),
           both / (lds + shf), both / (lds > shf ? lds : shf));
    return 0;
}
