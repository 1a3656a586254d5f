// FP64 pipe peak microbenchmark for the roofline denominator (MEASURED_PEAKS.json has no
// FP64 entry).  Each thread runs CH independent DFMA (or DADD) chains; the grid is
// SMs x BPS blocks of 256 threads.  Several (CH, BPS) shapes are timed and the best is
// reported, so the DFMA figure is a saturated pipe, not a latency-bound loop (round 1's
// 8-chain loop sustained 58.7 DFMA/clk/SM against 63.8 for DADD).  Also reports the nominal
// peak 2 * 64 DFMA/clk/SM * SMs * max clock.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void dadd_loop(double* out, int iters, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int c = 0; c < CH; ++c) x[c] = x[c] + b;
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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

template <class K>
float best_ms(K launch, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

template <int CH>
void shape(int sms, int bps, double* out, double& fma_rate, double& add_rate, int& best_ch, int& best_bps) {
    const int threads = 256, blocks = sms * bps;
    const int iters = 32768 / CH;  // same op count per thread for every CH
    const double n = double(blocks) * threads * iters * 8 * CH;
    const float mf = best_ms([&] { dfma_loop<CH><<<blocks, threads>>>(out, iters, 0.999999, 1e-9); }, 5);
    const float ma = best_ms([&] { dadd_loop<CH><<<blocks, threads>>>(out, iters, 1e-9); }, 5);
    if (n / (mf * 1e-3) > fma_rate) {
        fma_rate = n / (mf * 1e-3);
        best_ch = CH;
        best_bps = bps;
    }
    if (n / (ma * 1e-3) > add_rate) add_rate = n / (ma * 1e-3);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    cudaMalloc(&cyc, sizeof(long long));
    double fma_rate = 0, add_rate = 0;
    int best_ch = 0, best_bps = 0;
    for (int bps : {4, 8}) {
        shape<8>(sms, bps, out, fma_rate, add_rate, best_ch, best_bps);
        shape<16>(sms, bps, out, fma_rate, add_rate, best_ch, best_bps);
        shape<24>(sms, bps, out, fma_rate, add_rate, best_ch, best_bps);
        shape<32>(sms, bps, out, fma_rate, add_rate, best_ch, best_bps);
    }
    dfma_latency<<<1, 32>>>(out, cyc, 1024, 0.999999, 1e-9);
    long long hc;
    cudaMemcpy(&hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double nominal = 2.0 * 64 * sms * (clk_khz * 1e3) / 1e12;
    printf("{\"device\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.3f, \"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, "
           "\"dfma_per_clk_per_sm_at_max\": %.2f, \"dadd_per_clk_per_sm_at_max\": %.2f, \"best_chains\": %d, "
           "\"best_blocks_per_sm\": %d, \"dfma_dep_latency_cycles\": %.2f, \"max_clock_mhz\": %d, "
           "\"nominal_tflops\": %.3f}\n",
           p.name, sms, 2.0 * fma_rate / 1e12, fma_rate, add_rate, fma_rate / sms / (clk_khz * 1e3),
           add_rate / sms / (clk_khz * 1e3), best_ch, best_bps, double(hc) / (1024.0 * 16), clk_khz / 1000, nominal);
    return 0;
}
