// FP64 pipe peak microbenchmark for the roofline denominator (MEASURED_PEAKS.json has
// no FP64 entry).  Each thread runs 8 independent DFMA chains; grid = SMs x 8 blocks.
// Prints one JSON line: {"dfma_tflops": ..., "sm_clock_mhz_est": ..., ...}
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dadd_loop(double* out, int iters, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = x0 + b; x1 = x1 + b; x2 = x2 + b; x3 = x3 + b; x4 = x4 + b; x5 = x5 + b; x6 = x6 + b; x7 = x7 + b;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// single-warp dependent chain: latency
__global__ void dfma_latency(double* out, long long* cycles, int iters, double a, double b) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cycles = t1 - t0;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    cudaMalloc(&cyc, sizeof(long long));
    const int iters = 4096, threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best_fma = 1e30f, best_add = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_fma) best_fma = ms;
        cudaEventRecord(e0);
        dadd_loop<<<blocks, threads>>>(out, iters, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_add) best_add = ms;
    }
    const double n_fma = double(blocks) * threads * iters * 16 * 8;
    dfma_latency<<<1, 32>>>(out, cyc, 1024, 0.999999, 1e-9);
    long long hc;
    cudaMemcpy(&hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.3f, \"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, "
           "\"dfma_per_clk_per_sm_at_max\": %.2f, \"dfma_dep_latency_cycles\": %.2f, \"max_clock_mhz\": %d}\n",
           p.name, sms, 2.0 * n_fma / (best_fma * 1e-3) / 1e12, n_fma / (best_fma * 1e-3),
           n_fma / (best_add * 1e-3), n_fma / (best_fma * 1e-3) / sms / (clk_khz * 1e3),
           double(hc) / (1024.0 * 16), clk_khz / 1000);
    return 0;
}
