// Probe of the tcgen05.st 16x32bx2 lane/column mapping (development aid): each thread t
// stores 4 registers t*100 + r with one 16x32bx2.x4 store at lane 0 / column 0 and a half
// split offset of 8 columns, then every lane of the quadrant reads its 16 columns back.
#include <cstdio>
#include <cstdint>

__global__ void probe(uint32_t* out) {
    __shared__ uint32_t base;
    if (threadIdx.x < 32)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&base)))
                     : "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t t = threadIdx.x;
    // zero the 16 columns of every lane first
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(base),
                 "r"(0u));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.st.sync.aligned.16x32bx2.x4.b32 [%0], 8, {%1, %2, %3, %4};\n" ::"r"(base), "r"(t * 100),
                 "r"(t * 100 + 1), "r"(t * 100 + 2), "r"(t * 100 + 3));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(base));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int k = 0; k < 16; ++k) out[t * 16 + k] = r[k];
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(base) : "memory");
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 32 * 16 * 4);
    probe<<<1, 32>>>(d);
    uint32_t h[32 * 16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    for (int l = 0; l < 32; ++l) {
        printf("lane %2d:", l);
        for (int k = 0; k < 16; ++k) printf(" %5u", h[l * 16 + k]);
        printf("\n");
    }
}
