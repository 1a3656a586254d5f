// H2D copy rate from pinned staging right after host threads wrote it (development probe).
// nvcc -O2 -o h2d_probe h2d_probe.cu -lpthread
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const size_t bytes = 17u << 20;
    double *h, *d;
    cudaHostAlloc(reinterpret_cast<void**>(&h), bytes, cudaHostAllocPortable);
    cudaMalloc(reinterpret_cast<void**>(&d), bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double* hw;
    cudaHostAlloc(reinterpret_cast<void**>(&hw), bytes, cudaHostAllocPortable | cudaHostAllocWriteCombined);
    double* hp = h;
    for (int mode = 0; mode < 6; ++mode)
        for (int rep = 0; rep < 3; ++rep) {
            const int nt = mode == 5 ? 1 : 16, parts = mode == 2 ? 32 : 4;
            h = mode == 3 ? hw : hp;  // mode 3: write-combined staging; 4: non-temporal stores; 5: one writer thread
            if (mode >= 1) {  // host threads rewrite the buffer first
                std::vector<std::thread> th;
                for (int t = 0; t < nt; ++t)
                    th.emplace_back([&, t] {
                        const size_t n = bytes / 8 / nt;
                        if (mode == 4)
                            for (size_t i = 0; i < n; ++i) _mm_stream_si64(reinterpret_cast<long long*>(&h[t * n + i]), static_cast<long long>(i + rep));
                        else
                            if (mode == 4)
                            for (size_t i = 0; i < n; ++i) _mm_stream_si64(reinterpret_cast<long long*>(&h[t * n + i]), static_cast<long long>(i + rep));
                        else
                            for (size_t i = 0; i < n; ++i) h[t * n + i] = static_cast<double>(i + rep);
                    });
                for (auto& t : th) t.join();
            }
            const auto t0 = std::chrono::steady_clock::now();
            cudaEventRecord(e0, st);
            for (int p = 0; p < parts; ++p)
                cudaMemcpyAsync(reinterpret_cast<char*>(d) + bytes / parts * p, reinterpret_cast<char*>(h) + bytes / parts * p,
                                bytes / parts, cudaMemcpyHostToDevice, st);
            cudaEventRecord(e1, st);
            const auto t1 = std::chrono::steady_clock::now();
            cudaStreamSynchronize(st);
            const auto t2 = std::chrono::steady_clock::now();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::printf("mode %d (%s, %d copies): events %.3f ms = %.1f GB/s; enqueue %.3f ms, sync %.3f ms\n", mode,
                        mode ? "after host writes" : "untouched", parts, ms, bytes / ms / 1e6,
                        std::chrono::duration<double, std::milli>(t1 - t0).count(),
                        std::chrono::duration<double, std::milli>(t2 - t1).count());
        }
    return 0;
}
