// SASS probes of the engine's arithmetic primitives (one call per kernel, operands from
// global memory so nothing folds).  tools/flops_model.py compiles this for sm_100a,
// counts the FP64 instructions of each kernel and builds the per-term flop model.
#include "../../paper_2009_01177_b200/csrc/arith.cuh"

using namespace tor;

// every accumulator word reaches memory (differences of probes cancel these adds)
__device__ double sink(const Acc<double>& a) { return a.s.hi + a.s.lo + a.abs_sum; }
__device__ double sink(const Acc<dd>& a) { return a.s.hi + a.s.lo + a.h + a.c + a.abs_sum; }
__device__ double sink(const Acc<qd>& a) {
    return a.s.x[0] + a.s.x[1] + a.s.x[2] + a.s.x[3] + a.b0 + a.b1 + a.b2 + a.b3 + a.abs_sum;
}

#define PROBES(T, NAME)                                                                        \
    extern "C" __global__ void rank2_##NAME(const T* in, T* out) {                            \
        const int i = threadIdx.x;                                                             \
        out[i] = Arith<T>::rank2(in[i], in[i + 32], in[i + 64], in[i + 96], in[i + 128]);     \
    }                                                                                          \
    extern "C" __global__ void vec_##NAME(const T* in, T* out) {                              \
        const int i = threadIdx.x;                                                             \
        const T u = Arith<T>::mul(in[i], in[i + 32]);                                          \
        out[i] = u;                                                                            \
        out[i + 32] = Arith<T>::mul(Arith<T>::rank1s(in[i + 64], in[i + 96], u), in[i + 128]); \
    }                                                                                          \
    extern "C" __global__ void pivot_##NAME(const T* in, T* out, int* flags) {                \
        const int i = threadIdx.x;                                                             \
        const Piv<T> p = pivot2<T>(in[i], in[i + 32], in[i + 64], in[i + 96]);                 \
        out[i] = p.r1;                                                                         \
        out[i + 32] = p.u1;                                                                    \
        out[i + 64] = p.r2;                                                                    \
        out[i + 96] = p.tn;                                                                    \
        flags[i] = p.bad0 | (p.bad1 << 1);                                                     \
    }                                                                                          \
    extern "C" __global__ void leaf_##NAME(const T* in, T* out, int* flags) {                 \
        const int i = threadIdx.x;                                                             \
        bool bad;                                                                              \
        out[i] = leaf_term<T>(in[i], in[i + 32], in[i + 64], in[i + 96], bad);                 \
        flags[i] = bad;                                                                        \
    }                                                                                          \
    extern "C" __global__ void accadd1_##NAME(const T* in, double* out, const int* z) {        \
        const int i = threadIdx.x;                                                             \
        Acc<T> a;                                                                              \
        a.add(in[i], z[i] & 1, z[i] >> 1);                                                     \
        out[i] = sink(a);                                                                      \
    }                                                                                          \
    extern "C" __global__ void accadd2_##NAME(const T* in, double* out, const int* z) {        \
        const int i = threadIdx.x;                                                             \
        Acc<T> a;                                                                              \
        a.add(in[i], z[i] & 1, z[i] >> 1);                                                     \
        a.add(in[i + 32], z[i] & 2, z[i] >> 2);                                                \
        out[i] = sink(a);                                                                      \
    }                                                                                          \
    extern "C" __global__ void accflush_##NAME(const T* in, double* out, const int* z) {       \
        const int i = threadIdx.x;                                                             \
        Acc<T> a;                                                                              \
        a.add(in[i], z[i] & 1, z[i] >> 1);                                                     \
        a.add(in[i + 32], z[i] & 2, z[i] >> 2);                                                \
        a.flush();                                                                             \
        out[i] = sink(a);                                                                      \
    }

PROBES(double, fp64)
PROBES(dd, dd)
PROBES(qd, qd)

// QD building blocks (for the QD cost breakdown)
extern "C" __global__ void mul_qd(const qd* in, qd* out) {
    const int i = threadIdx.x;
    out[i] = qd_mul(in[i], in[i + 32]);
}
extern "C" __global__ void add_qd(const qd* in, qd* out) {
    const int i = threadIdx.x;
    out[i] = qd_add(in[i], in[i + 32]);
}
extern "C" __global__ void rsqrt_qd(const qd* in, qd* out) {
    const int i = threadIdx.x;
    out[i] = qd_rsqrt(in[i]);
}
