// sm_100a kernels of the Torontonian engine (see engine.cuh and DESIGN.md).
//
// Work decomposition of the 2^n subsets (binary decision tree over modes 0..n-1,
// decision "include mode m" = Cholesky elimination of the mode's 2x2 pair block
// from the current Schur complement; "exclude" = drop the pair, a view):
//
//   depth 0 .. c           prefix levels, level-synchronous in global memory
//                          (prefix_level_kernel, one warp per include node)
//   depth c                jobs: 2^c prefix classes (top c reference-mask bits),
//                          one warp per job (subtree_kernel)
//   depth c .. n-q0        warp DFS, warp-cooperative eliminations, per-warp
//                          global scratch stack (L1/L2 resident)
//   depth n-q0 .. n-L      5-level breadth-first fan-out in shared memory, one
//                          node per lane at the end (32 lanes)
//   depth n-L .. n         per-lane register-resident subtree (fully unrolled)
//
// Every include node emits one signed term t = 1/sqrt(det R_Z) = prod of pivot
// rsqrts; terms accumulate per lane (compensated), lanes fold by a fixed xor
// butterfly, jobs by a fixed binary tree: the result is bit-identical for any
// grid size, SM count or power-of-two shard count.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "arith.cuh"
#include "engine.cuh"

namespace tor {

namespace {

constexpr int FAN = 5;  // breadth-first fan-out levels -> 32 lane nodes
constexpr int MAX_LEVELS = 48;
// job states have <= kMaxJobModes modes: the prefix depth is c >= n - kMaxJobModes, and 32
// keeps the prefix levels of an n = 50 shard (the paper's case) within a few GB
constexpr int kMaxJobModes = 32;
constexpr uint64_t kWantJobs = 262144;
#ifndef TOR_WANT_JOBS_BATCH
#define TOR_WANT_JOBS_BATCH 32768  // cfg3 4096 x n=16: fp64 2.19 -> 1.95 ms, DD 5.59 -> 5.47 (262144 / 65536 / 32768 / 8192 measured)
#endif
constexpr uint64_t kWantJobsBatch = TOR_WANT_JOBS_BATCH;  // batches of several instances
constexpr int kShardBits = 6;
#ifndef TOR_MB_HINT
#define TOR_MB_HINT 100  // mbarrier try_wait suspend-time hint (ns): 1e6 measured 0.3% slower
#endif


__host__ __device__ constexpr int tri_sz(int d) { return d * (d + 1) / 2; }
__host__ __device__ __forceinline__ int tri_ix(int d, int i, int j) {
    return i * d - ((i * (i + 1)) >> 1) + j;
}
// A view that drops the first s rows of a packed D-row triangle is itself a packed
// (D-s)-row triangle stored contiguously at tri_ix(D, s, s):
//   tri_ix(D, s+a, s+b) = tri_ix(D, s, s) + tri_ix(D-s, a, b).
// So every node state (and every trailing block) is addressed as (pointer, dim).

// Rank-2 trailing update of an elimination from a q-mode state (m = 2q rows): child
// entry k (packed (m-2)-row triangle) reads parent entry 2m-1+k and the pivot-row
// vectors at rows 2+i, 2+j.  (i,j) tables hold (2+i) | (2+j) << 16.
__host__ __device__ constexpr uint32_t ij_word(int i, int j) {
    return static_cast<uint32_t>(2 + i) | (static_cast<uint32_t>(2 + j) << 16);
}
// DFS tables in global memory: dims 2a, a = 1 .. kMaxJobModes-1, table a at ijtab_off(a)
__host__ __device__ constexpr int ijtab_off(int a) { return 2 * (a - 1) * a * (2 * a - 1) / 6 + (a - 1) * a / 2; }

// Lane-level register depth per word type (register budget: the L-mode state is
// read from shared memory, states of < L modes live in registers).
// TMEM: the lane states of the last fan-out level are handed to their lanes through
// tensor memory (each lane's own TMEM row) instead of shared-memory buffers; needs
// 4-warp CTAs (one warp per TMEM lane quadrant).
template <class T> struct Cfg;
template <> struct Cfg<double> {
    // unspecialised: every warp runs whole leaves, lane subtrees of 5 modes from shared memory.
    // (The DD kernel's structure with 8-byte words -- 4 producers + 8 consumers, level 5 and
    // L = 4 lane subtrees in TMEM -- measured slower on config 3: 2.96 ms with the producers
    // running level 1 only, 3.25 with levels 1-2, vs 2.51: the producers' job-state loads
    // bound it and the consumers' fp64 lane subtrees are too short to hide them.)
#ifndef TOR_F64_MINB
#define TOR_F64_MINB 1
#endif
#ifndef TOR_F64_L
#define TOR_F64_L 5
#endif
    static constexpr int L = TOR_F64_L;
    static constexpr int WPB = 4;
    static constexpr int MINB = TOR_F64_MINB;
    static constexpr bool TMEM = false;
    static constexpr bool WS = false;
    static constexpr int WS_MODE = 0;
    static constexpr bool TSHARE = false;
};
template <> struct Cfg<dd> {
    static constexpr int L = 4;
    // Warp specialisation (WS_MODE 2; the other types run unspecialised, WS_MODE 0):
    // 4 producers (DFS + fan-out levels 1-2) + 8 consumers (levels 3-5 + lane subtrees),
    // each producer alternating between two jobs / two consumers; one 12-warp CTA per SM
    // at 168 registers (3 warps per SM sub-partition), two consumers per TMEM lane quadrant
    // (256 columns each)
    static constexpr int WS_MODE = 2;
    static constexpr bool WS = true;
    static constexpr int WPB = 12;
    static constexpr int MINB = 1;
    static constexpr bool TMEM = true;
    static constexpr bool TSHARE = false;
};
template <> struct Cfg<qd> {
#ifndef TOR_QD_L
#define TOR_QD_L 3
#endif
#ifndef TOR_QD_MINB
#define TOR_QD_MINB 1
#endif
    static constexpr int L = TOR_QD_L;
    // Time-shared areas (TSHARE): a QD warp area is ~50 KB, so only four fit on an SM.  Two warps
    // (w, w + 4: same SM sub-partition, same TMEM lane quadrant) take turns on one area: a warp
    // runs the DFS step and the fan-out of its leaf in the area, copies the 32 lane-node states
    // into its own TMEM columns (21 entries x 8 words per lane), hands the area to its partner
    // and runs the lane subtrees from TMEM -- 8 warps per SM instead of 4, same per-job
    // arithmetic and order (bit-identical results).
    // (one warp per CTA, four CTAs per SM: n = 28 82.9 ms against 72.4)
    static constexpr bool TSHARE = true;
    static constexpr int WPB = 8;
    static constexpr int MINB = TOR_QD_MINB;
    static constexpr bool TMEM = false;
    static constexpr bool WS = false;
    static constexpr int WS_MODE = 0;
};

template <class T> constexpr int root_modes() { return Cfg<T>::L + FAN; }

// WS mode 2: first fan-out level run by the consumer warps (the producers run the DFS
// and levels 1 .. cons_first - 1)
#ifndef TOR_CONS_FIRST
#define TOR_CONS_FIRST 3
#endif
template <class T> __host__ __device__ constexpr int cons_first() { return TOR_CONS_FIRST; }

constexpr int kIjTabEntries = ijtab_off(kMaxJobModes);
__device__ uint32_t g_ijtab[kIjTabEntries];

// ----------------------------------------------------------------- jobs ----
template <class T> struct Job {
    const T* base;  // buffer holding the node's state (packed triangle, `dim` rows)
    int dim;        // rows of the buffer
    int skip;       // leading modes of the buffer dropped (excluded) for this node
    int inst;       // instance index
    int nsel;       // |Z| so far
    uint64_t mask;  // reference-convention mask bits of the node's subset
    T t;            // 1/sqrt(det R_Z)
};

struct PrefixGeom {
    int n;                             // modes
    int c;                             // prefix depth
    size_t off[MAX_LEVELS + 1];        // entry offset of level e buffers (per instance)
    size_t toff[MAX_LEVELS + 1];       // offset of level e t values (per instance)
    uint64_t plo[MAX_LEVELS + 1];      // level e stores include nodes p = plo[e] .. (compact: a
                                       // shard keeps only the nodes under its class range)
    size_t inst_entries;               // entries per instance
    size_t inst_ts;                    // t values per instance
};

__device__ __forceinline__ void report_breakdown(unsigned long long* err, uint64_t mask, int row) {
    // smallest failing mask wins (deterministic); row in the low byte
    atomicMin(err, (static_cast<unsigned long long>(mask) << 8) | static_cast<unsigned long long>(row & 0xff));
}
// Per-thread breakdown sink of the lane-level code: the same min key kept in a register
// and published once per warp lifetime (flush), so the pivot checks are selects instead
// of branches around an atomic (no basic-block split between consecutive pivot chains).
struct LocalErr {
    unsigned long long v = ~0ull;
    __device__ __forceinline__ void flush(unsigned long long* err) const {
        if (v != ~0ull) atomicMin(err, v);
    }
};
__device__ __forceinline__ void report_breakdown(LocalErr* err, uint64_t mask, int row) {
    const unsigned long long key = (static_cast<unsigned long long>(mask) << 8) | static_cast<unsigned long long>(row & 0xff);
    err->v = key < err->v ? key : err->v;
}

template <class T> __device__ __forceinline__ T shfl_xor_t(const T& v, int m);
template <> __device__ __forceinline__ double shfl_xor_t<double>(const double& v, int m) {
    return __shfl_xor_sync(0xffffffffu, v, m);
}
template <> __device__ __forceinline__ dd shfl_xor_t<dd>(const dd& v, int m) {
    return dd{__shfl_xor_sync(0xffffffffu, v.hi, m), __shfl_xor_sync(0xffffffffu, v.lo, m)};
}
template <> __device__ __forceinline__ qd shfl_xor_t<qd>(const qd& v, int m) {
    qd r;
#pragma unroll
    for (int i = 0; i < 4; ++i) r.x[i] = __shfl_xor_sync(0xffffffffu, v.x[i], m);
    return r;
}
template <class T> __device__ __forceinline__ T shfl_t(const T& v, int src);
template <> __device__ __forceinline__ double shfl_t<double>(const double& v, int s) {
    return __shfl_sync(0xffffffffu, v, s);
}
template <> __device__ __forceinline__ dd shfl_t<dd>(const dd& v, int s) {
    return dd{__shfl_sync(0xffffffffu, v.hi, s), __shfl_sync(0xffffffffu, v.lo, s)};
}
template <> __device__ __forceinline__ qd shfl_t<qd>(const qd& v, int s) {
    qd r;
#pragma unroll
    for (int i = 0; i < 4; ++i) r.x[i] = __shfl_sync(0xffffffffu, v.x[i], s);
    return r;
}

// (fp64 mode accumulates in DD: a.s is a dd there)
template <class AC> __device__ __forceinline__ void warp_fold(AC& a) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        AC o;
        o.s = shfl_xor_t(a.s, m);
        o.abs_sum = __shfl_xor_sync(0xffffffffu, a.abs_sum, m);
        a.merge(o);
    }
}



// ------------------------------------------------ warp-cooperative elimination --
// Eliminates the first mode (rows 0,1) of the q-mode view (S, d, sr) into the
// packed (2q-2)-row triangle dst; t_out = t * rho1 * rho2.  uw: shared scratch of
// 4q entries.  All lanes compute the pivot chain redundantly (warp-uniform).  The
// trailing entries [kbeg, kend) are this warp's share (several warps may split one
// elimination: each recomputes the pivots and vectors, only part 0 writes t_out and
// reports breakdowns).
template <class T>
__device__ void warp_elim(const T* S, int d, int sr, int q, T* dst, const T& t_in, T* t_out, T* uw,
                          uint64_t mask, int nsel, unsigned long long* err, int part = 0, int nparts = 1) {
    using A = Arith<T>;
    const int lane = threadIdx.x & 31;
    const Piv<T> pv = pivot2<T>(S[tri_ix(d, sr, sr)], S[tri_ix(d, sr, sr + 1)], S[tri_ix(d, sr + 1, sr + 1)], t_in);
    const T r1 = pv.r1, u1 = pv.u1, r2 = pv.r2;
    if (lane == 0 && part == 0) {
        if (pv.bad0 || pv.bad1) report_breakdown(err, mask, 2 * nsel + (pv.bad0 ? 0 : 1));
        *t_out = pv.tn;
    }
    const int m = 2 * q;
    for (int j = 2 + lane; j < m; j += 32) {
        T uj, wj;
        A::vec(S[tri_ix(d, sr, sr + j)], S[tri_ix(d, sr + 1, sr + j)], r1, u1, r2, uj, wj);
        uw[j] = uj;
        uw[m + j] = wj;
    }
    __syncwarp();
    // trailing update: 4 entries per lane per round, loads issued together so the
    // (L2-resident) source reads overlap; positions advance incrementally.
    const int dn = m - 2;
    const int total = tri_sz(dn);
    const int per = ((total + nparts - 1) / nparts + 127) & ~127;
    const int kbeg = part * per, kend = min(total, kbeg + per);
    int i = 0, k0 = kbeg + lane;
    while (i < dn && k0 >= dn - i) {
        k0 -= dn - i;
        ++i;
    }
    int j = i + k0;
    for (int kb = kbeg; kb < kend; kb += 128) {
        int ii[4], jj[4];
        T sv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool ok = kb + lane + 32 * u < kend;
            ii[u] = ok ? i : 0;
            jj[u] = ok ? j : 0;
            sv[u] = S[tri_ix(d, sr + 2 + ii[u], sr + 2 + jj[u])];
            j += 32;
            while (i < dn && j >= dn) {
                j -= dn - (i + 1);
                ++i;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const T v = A::rank2(sv[u], uw[2 + ii[u]], uw[2 + jj[u]], uw[m + 2 + ii[u]], uw[m + 2 + jj[u]]);
            const int k = kb + lane + 32 * u;
            if (k < kend) dst[k] = v;
        }
    }
    __syncwarp();
}


// DFS step of the subtree kernel: eliminates the first mode of the q-mode source
// state P (contiguous packed 2q-row triangle, HBM/L2 resident) and writes (a) the new
// (q-1)-mode state to its DFS slot (only when later leaves read it) and (b) its
// trailing Q0 modes -- the contiguous tail of the new state -- straight into the
// shared-memory root of the leaf that follows.  Entry k of the new state reads P at
// 2m-1+k; its (i,j) comes from the global table tb.  All loads of the first batch
// are issued before the pivot chain: one L2 round trip.
template <class T, int Q0>
__device__ void dfs_elim(const T* P, int q, T* slot, bool write_slot, T* root, const T& t_in, T* t_out, T* uw,
                         const uint32_t* tb, uint64_t mask, int nsel, unsigned long long* err) {
    using A = Arith<T>;
#ifndef TOR_NB
#define TOR_NB 6
#endif

#ifndef TOR_QD_NB
#define TOR_QD_NB 2
#endif
    constexpr int NB = sizeof(T) == sizeof(qd) ? TOR_QD_NB : TOR_NB;  // entries per lane per batch
    constexpr int RT = tri_sz(2 * Q0);
    const int lane = threadIdx.x & 31;
    const int m = 2 * q;
    const int total = tri_sz(m - 2);
    const T* Pt = P + 2 * m - 1;
    // ---- issue loads: pivot block, this lane's pivot-row entries, first entry batch
    const T p00 = P[0], p01 = P[1], p11 = P[m];
    T v0[2], v1[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int j = 2 + lane + 32 * r;
        const int jc = j < m ? j : m - 1;
        v0[r] = P[jc];
        v1[r] = P[m - 1 + jc];
    }
    uint32_t ij[NB];
    T sv[NB];
    auto load_batch = [&](int kb) {
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int k = kb + lane + 32 * u;
            const int kc = k < total ? k : total - 1;
            sv[u] = Pt[kc];
            ij[u] = __ldg(tb + kc);
        }
    };
    load_batch(0);
    // ---- pivots (all lanes, warp-uniform) and pivot-row vectors
    const Piv<T> pv = pivot2_shared<T>(p00, p01, p11, t_in, lane, 1);
    if (lane == 0) {
        if (pv.bad0 || pv.bad1) report_breakdown(err, mask, 2 * nsel + (pv.bad0 ? 0 : 1));
        *t_out = pv.tn;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int jv = 2 + lane + 32 * r;
        if (jv < m) {
            T uj, wj;
            A::vec(v0[r], v1[r], pv.r1, pv.u1, pv.r2, uj, wj);
            uw[jv] = uj;
            uw[m + jv] = wj;
        }
    }
    __syncwarp();
    // ---- trailing update, batch by batch
    T* rootb = root - (total - RT);  // entry k >= total-RT is root entry k-(total-RT)
    // (a second register set holding the next batch's L2 loads in flight measured slower:
    // n = 32 DD 84.5 vs 82.5 ms, 168 registers)
    for (int kb = 0;;) {
        T out[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int i = static_cast<int>(ij[u] & 0xffffu), j = static_cast<int>(ij[u] >> 16);
            out[u] = A::rank2(sv[u], uw[i], uw[j], uw[m + i], uw[m + j]);
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int k = kb + lane + 32 * u;
            if (k < total) {
                if (write_slot) slot[k] = out[u];
                if (k >= total - RT) rootb[k] = out[u];
            }
        }
        kb += 32 * NB;
        if (kb >= total) break;
        load_batch(kb);
    }
    __syncwarp();
}

// ---------------------------------------------------------- prefix levels ----
template <class T>
__device__ __forceinline__ void node_view(const PrefixGeom& g, const T* pool, const T* tpool, int inst, int e,
                                          uint64_t c, const T*& base, int& dim, int& skip, T& t) {
    const T* ib = pool + inst * g.inst_entries;
    if (c == 0) {
        base = ib + g.off[0];
        dim = 2 * g.n;
        skip = e;
        t = Arith<T>::one();
        return;
    }
    const int tz = __ffsll(static_cast<long long>(c)) - 1;
    const int lvl = e - tz;
    const uint64_t p = (c >> tz) >> 1;
    dim = 2 * (g.n - lvl);
    base = ib + g.off[lvl] + (p - g.plo[lvl]) * static_cast<uint64_t>(tri_sz(dim));
    skip = tz;
    t = tpool[inst * g.inst_ts + g.toff[lvl] + (p - g.plo[lvl])];
}

// Level e: every include node (inst, p), p in [plo, plo + cnt), eliminates the first
// mode of its parent view (e-1, p) into level-e buffer p; `parts` warps share one
// elimination (top levels: few nodes, long trailing updates).
template <class T>
__global__ void prefix_level_kernel(PrefixGeom g, T* pool, T* tpool, int e, int ninst, uint64_t plo, uint64_t cnt,
                                    int parts, unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* uw_all = reinterpret_cast<T*>(smem_raw);
    const int wib = threadIdx.x >> 5;
    T* uw = uw_all + wib * (4 * g.n);
    const uint64_t total = cnt * ninst * parts;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t it = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < total; it += nw) {
        const int part = static_cast<int>(it % parts);
        const uint64_t node = it / parts;
        const int inst = static_cast<int>(node / cnt);
        const uint64_t p = plo + node % cnt;
        const T* base;
        int dim, skip;
        T t;
        node_view<T>(g, pool, tpool, inst, e - 1, p, base, dim, skip, t);
        const int q = g.n - (e - 1);
        T* dst = pool + inst * g.inst_entries + g.off[e] + (p - g.plo[e]) * static_cast<uint64_t>(tri_sz(2 * (g.n - e)));
        T* tdst = tpool + inst * g.inst_ts + g.toff[e] + (p - g.plo[e]);
        const uint64_t mask = ((p << 1) | 1ull) << (g.n - e);
        warp_elim<T>(base, dim, 2 * skip, q, dst, t, tdst, uw, mask, __popcll(mask) - 1, err, part, parts);
    }
}

template <class T>
__global__ void make_jobs_kernel(PrefixGeom g, const T* pool, const T* tpool, int ninst, uint64_t lo,
                                 uint64_t hi, Job<T>* jobs) {
    const uint64_t per = hi - lo;
    const uint64_t total = per * ninst;
    for (uint64_t it = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; it < total;
         it += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int inst = static_cast<int>(it / per);
        const uint64_t c = lo + it % per;
        Job<T> J;
        node_view<T>(g, pool, tpool, inst, g.c, c, J.base, J.dim, J.skip, J.t);
        J.inst = inst;
        J.mask = g.c ? (c << (g.n - g.c)) : 0;
        J.nsel = __popcll(c);
        jobs[it] = J;
    }
}

// Direct prefix for slices with class bits beyond the materialised prefix depth:
// one warp per class walks modes 0..k-1 (include -> eliminate into the class's own
// ping-pong buffers, exclude -> skip).
template <class T>
__global__ void direct_prefix_kernel(int n, int k, const T* R, int ninst, size_t inst_entries, uint64_t lo,
                                     uint64_t hi, T* work, size_t work_stride, Job<T>* jobs,
                                     unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* uw_all = reinterpret_cast<T*>(smem_raw);
    T* tslot = uw_all + (blockDim.x >> 5) * (4 * n);
    const int wib = threadIdx.x >> 5;
    T* uw = uw_all + wib * (4 * n);
    T* tt = tslot + wib;
    const int lane = threadIdx.x & 31;
    const uint64_t per = hi - lo;
    const uint64_t total = per * ninst;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t it = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < total; it += nw) {
        const int inst = static_cast<int>(it / per);
        const uint64_t cls = lo + it % per;
        const T* base = R + inst * inst_entries;
        int dim = 2 * n, skip = 0, nsel = 0;
        T t = Arith<T>::one();
        T* bufs[2] = {work + it * work_stride, work + it * work_stride + tri_sz(2 * n)};
        int cur = 0;
        uint64_t mask = 0;
        for (int m = 0; m < k; ++m) {
            const bool inc = (cls >> (k - 1 - m)) & 1;
            if (!inc) {
                ++skip;
                continue;
            }
            mask |= 1ull << (n - 1 - m);
            const int q = dim / 2 - skip;
            T* dst = bufs[cur];
            warp_elim<T>(base, dim, 2 * skip, q, dst, t, tt, uw, mask, nsel, err);
            __syncwarp();
            t = *tt;
            __syncwarp();
            base = dst;
            dim = 2 * (q - 1);
            skip = 0;
            cur ^= 1;
            ++nsel;
        }
        if (lane == 0) {
            Job<T> J;
            J.base = base;
            J.dim = dim;
            J.skip = skip;
            J.inst = inst;
            J.nsel = nsel;
            J.mask = mask;
            J.t = t;
            jobs[it] = J;
        }
        __syncwarp();
    }
}

// ------------------------------------------------ register-level subtrees ----
// State of Q modes in registers: packed upper triangle of 2Q rows.
// Pivot chain inside the lane subtrees: optionally one out-of-line copy (instruction
// footprint) instead of one per call site.
template <class T>
__device__ __forceinline__ Piv<T> piv_lt(const T& s00, const T& s01, const T& s11, const T& t) {
    return pivot2<T>(s00, s01, s11, t);
}

template <class T, int Q> struct St {
    T e[tri_sz(2 * Q)];
};

template <int D> __device__ __forceinline__ constexpr int cix(int i, int j) { return i * D - (i * (i + 1)) / 2 + j; }

// Eliminate mode 0 of a Q-mode register state into a (Q-1)-mode state.
template <class T, int Q, class E>
__device__ __forceinline__ void elim_reg(const St<T, Q>& S, St<T, Q - 1>& out, const T& t, T& tout, uint64_t mask,
                                         int nsel, E* err) {
    using A = Arith<T>;
    constexpr int M = 2 * Q;
    const Piv<T> pv = piv_lt<T>(S.e[cix<M>(0, 0)], S.e[cix<M>(0, 1)], S.e[cix<M>(1, 1)], t);
    const T r1 = pv.r1, u1 = pv.u1, r2 = pv.r2;
    if (pv.bad0 || pv.bad1) report_breakdown(err, mask, 2 * nsel + (pv.bad0 ? 0 : 1));
    tout = pv.tn;
    T u[M], w[M];
#pragma unroll
    for (int j = 2; j < M; ++j) {
        A::vec(S.e[cix<M>(0, j)], S.e[cix<M>(1, j)], r1, u1, r2, u[j], w[j]);
    }
#pragma unroll
    for (int i = 2; i < M; ++i)
#pragma unroll
        for (int j = i; j < M; ++j)
            out.e[cix<M - 2>(i - 2, j - 2)] = A::rank2(S.e[cix<M>(i, j)], u[i], u[j], w[i], w[j]);
}

// All nonempty subsets of the Q register modes (the node's own term excluded).
// neg: sign of the current node's term; bits: reference mask of the node.
// Levels with Q >= kLoopQ run their include/exclude branches as a 2-trip loop so
// the subtree below is emitted once (instruction-cache footprint grows with L, not
// 2^L); lower levels stay fully unrolled for instruction-level parallelism.
#ifndef TOR_LOOPQ
#define TOR_LOOPQ 3
#endif
constexpr int kLoopQ = TOR_LOOPQ;
#ifndef TOR_QD_LOOPQ
#define TOR_QD_LOOPQ 3
#endif
constexpr int kLoopQQd = TOR_QD_LOOPQ;
#ifndef TOR_F64_LOOPQ
#define TOR_F64_LOOPQ 4  // fp64: levels of >= 4 modes as loops (cfg3 fp64 2.50 -> 2.36 ms vs 3; 5: 2.36)
#endif
constexpr int kLoopQF64 = TOR_F64_LOOPQ;

template <class T, int Q> struct SubReg {
    template <class AC, class E>
    __device__ __forceinline__ static void branch(const St<T, Q>& S, int br, const T& t, bool neg, uint64_t mask,
                                                  int nsel, AC& acc, E* err) {
        constexpr int M = 2 * Q;
        const uint64_t bit = 1ull << (Q - 1);
        St<T, Q - 1> Sn;
        T tn;
        if (br == 0) {
            elim_reg<T, Q>(S, Sn, t, tn, mask | bit, nsel, err);
            acc.add(tn, !neg, nsel + 1);
        } else {
#pragma unroll
            for (int i = 2; i < M; ++i)
#pragma unroll
                for (int j = i; j < M; ++j) Sn.e[cix<M - 2>(i - 2, j - 2)] = S.e[cix<M>(i, j)];
            tn = t;
        }
        SubReg<T, Q - 1>::run(Sn, tn, br == 0 ? !neg : neg, br == 0 ? (mask | bit) : mask, nsel + (br == 0),
                              acc, err);
    }
    template <class AC, class E>
    __device__ __forceinline__ static void run(const St<T, Q>& S, const T& t, bool neg, uint64_t mask, int nsel,
                                               AC& acc, E* err) {
        if constexpr (Q >= (sizeof(T) == sizeof(qd) ? kLoopQQd : (sizeof(T) == sizeof(double) ? kLoopQF64 : kLoopQ))) {
#pragma unroll 1
            for (int br = 0; br < 2; ++br) branch(S, br, t, neg, mask, nsel, acc, err);
        } else {
            branch(S, 0, t, neg, mask, nsel, acc, err);
            branch(S, 1, t, neg, mask, nsel, acc, err);
        }
    }
};
template <class T> struct SubReg<T, 1> {
    template <class AC, class E>
    __device__ __forceinline__ static void run(const St<T, 1>& S, const T& t, bool neg, uint64_t mask, int nsel,
                                               AC& acc, E* err) {
        bool bad;
        const T tn = leaf_term<T>(S.e[0], S.e[1], S.e[2], t, bad);
        // both pivots of the last mode: a negative-definite 2x2 block has det > 0.  The state
        // word may be unnormalised (DD grid leading word a multiple of 2^-49, lazy QD words):
        // the sign comes from the word sum, not the leading word alone
        const bool bad0 = nonpositive(Arith<T>::sign_val(Arith<T>::unb(S.e[0])));
        if (bad || bad0) report_breakdown(err, mask | 1ull, 2 * nsel + (bad0 ? 0 : 1));
        acc.add(tn, !neg, nsel + 1);
    }
};

// Lane subtree rooted at an L-mode view in shared memory: emits the node's own
// term and all 2^L - 1 extensions.  Branch 0 includes the first view mode (its
// elimination reads shared memory), branch 1 excludes it (loads the trailing block).
template <class T, int L, class AC, class E, class View>
__device__ __forceinline__ void lane_tree_v(const View& V, const T& t, bool neg, uint64_t mask, int nsel, AC& acc,
                                            E* err) {
    using A = Arith<T>;
    constexpr int M = 2 * L;
    acc.add(t, neg, nsel);
    const uint64_t bit = 1ull << (L - 1);
    auto branch = [&](int br) {
        St<T, L - 1> Sn;
        T tn;
        if (br == 0) {
            const Piv<T> pv = pivot2<T>(V(0, 0), V(0, 1), V(1, 1), t);
            const T r1 = pv.r1, u1 = pv.u1, r2 = pv.r2;
            if (pv.bad0 || pv.bad1) report_breakdown(err, mask | bit, 2 * nsel + (pv.bad0 ? 0 : 1));
            tn = pv.tn;
            T u[M], w[M];
#pragma unroll
            for (int j = 2; j < M; ++j) {
                A::vec(V(0, j), V(1, j), r1, u1, r2, u[j], w[j]);
            }
#pragma unroll
            for (int i = 2; i < M; ++i)
#pragma unroll
                for (int j = i; j < M; ++j)
                    Sn.e[cix<M - 2>(i - 2, j - 2)] = A::rank2(V(i, j), u[i], u[j], w[i], w[j]);
            acc.add(tn, !neg, nsel + 1);
        } else {
#pragma unroll
            for (int i = 2; i < M; ++i)
#pragma unroll
                for (int j = i; j < M; ++j) Sn.e[cix<M - 2>(i - 2, j - 2)] = V(i, j);
            tn = t;
        }
        SubReg<T, L - 1>::run(Sn, tn, br == 0 ? !neg : neg, br == 0 ? (mask | bit) : mask, nsel + (br == 0), acc,
                              err);
    };
#pragma unroll 1
    for (int br = 0; br < 2; ++br) branch(br);
}
template <class T> struct SmemView;
template <class T, int L, class AC, class E>
__device__ __forceinline__ void lane_tree(const T* S, int d, int sr, const T& t, bool neg, uint64_t mask, int nsel,
                                          AC& acc, E* err) {
    lane_tree_v<T, L, AC, E>(SmemView<T>{S, d, sr}, t, neg, mask, nsel, acc, err);
}

// ------------------------------------------------------------------ TMEM ----
// Tensor memory as per-lane private storage: a warp w of a 4-warp CTA owns TMEM lanes
// 32(w%4)..+31; lane l's row holds its level-FAN state, entry k at columns 4k..4k+3.
__device__ __forceinline__ void tm_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void dd_to_u32(const dd& v, uint32_t* r) {
    r[0] = static_cast<uint32_t>(__double2loint(v.hi));
    r[1] = static_cast<uint32_t>(__double2hiint(v.hi));
    r[2] = static_cast<uint32_t>(__double2loint(v.lo));
    r[3] = static_cast<uint32_t>(__double2hiint(v.lo));
}
__device__ __forceinline__ dd u32_to_dd(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return dd{__hiloint2double(static_cast<int>(b), static_cast<int>(a)),
              __hiloint2double(static_cast<int>(d), static_cast<int>(c))};
}
// TMEM words of one state entry: U 32-bit columns (2 for fp64, 4 for DD)
template <class T> struct TmU {
    static constexpr int U = 2 * Arith<T>::K;
    static constexpr int EPL = 16 / U;  // entries per 16-column load / store
};
__device__ __forceinline__ void to_u32(const dd& v, uint32_t* r) { dd_to_u32(v, r); }
__device__ __forceinline__ void to_u32(const double& v, uint32_t* r) {
    r[0] = static_cast<uint32_t>(__double2loint(v));
    r[1] = static_cast<uint32_t>(__double2hiint(v));
}
template <class T> __device__ __forceinline__ T from_u32(const uint32_t* r);
template <> __device__ __forceinline__ dd from_u32<dd>(const uint32_t* r) { return u32_to_dd(r[0], r[1], r[2], r[3]); }
template <> __device__ __forceinline__ double from_u32<double>(const uint32_t* r) {
    return __hiloint2double(static_cast<int>(r[1]), static_cast<int>(r[0]));
}
__device__ __forceinline__ void to_u32(const qd& v, uint32_t* r) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r[2 * i] = static_cast<uint32_t>(__double2loint(v.x[i]));
        r[2 * i + 1] = static_cast<uint32_t>(__double2hiint(v.x[i]));
    }
}
template <> __device__ __forceinline__ qd from_u32<qd>(const uint32_t* r) {
    qd v;
#pragma unroll
    for (int i = 0; i < 4; ++i) v.x[i] = __hiloint2double(static_cast<int>(r[2 * i + 1]), static_cast<int>(r[2 * i]));
    return v;
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tm_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(a), "=r"(b) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
// one state entry (U words)
template <int U> __device__ __forceinline__ void tm_ld_e(uint32_t taddr, uint32_t* r) {
    if constexpr (U == 8) tm_ld8(taddr, r);
    else if constexpr (U == 4) tm_ld4(taddr, r[0], r[1], r[2], r[3]);
    else tm_ld2(taddr, r[0], r[1]);
}
template <int U> __device__ __forceinline__ void tm_st_e(uint32_t taddr, const uint32_t* r) {
    if constexpr (U == 8) tm_st8(taddr, r);
    else if constexpr (U == 4) tm_st4(taddr, r[0], r[1], r[2], r[3]);
    else tm_st2(taddr, r[0], r[1]);
}
// Lane-state accessors of lane_tree: entry (i, j) of the lane's D-row view from shared memory,
// or entry (i, j) of the lane's own TMEM row (natural layout, entry k at columns U k), loaded
// where it is used
template <class T> struct SmemView {
    const T* S;
    int d, sr;
    __device__ __forceinline__ T operator()(int i, int j) const { return S[tri_ix(d, sr + i, sr + j)]; }
};
template <class T, int D> struct TmemView {
    uint32_t row;
    __device__ __forceinline__ T operator()(int i, int j) const {
        uint32_t r[TmU<T>::U];
        tm_ld_e<TmU<T>::U>(row + static_cast<uint32_t>(TmU<T>::U * cix<D>(i, j)), r);
        tm_wait_ld();
        return from_u32<T>(r);
    }
};

// (row, col) of flat index k in a packed D-row upper triangle (compile-time)
__host__ __device__ constexpr int tri_row(int D, int k) {
    int i = 0;
    while (k >= D - i) {
        k -= D - i;
        ++i;
    }
    return i;
}
__host__ __device__ constexpr int tri_col(int D, int k) {
    int i = 0;
    while (k >= D - i) {
        k -= D - i;
        ++i;
    }
    return i + k;
}
// TMEM layout of a lane's level-FAN state (packed D = 2L row triangle, D = 8).  The
// level-FAN include child is formed by a thread pair (see FanLevel): entries with i + j < D-1
// ("A" set, 16 entries, row-major order A[0..15]) by one thread, their mirrors
// (D-1-j, D-1-i) by the other, the 4 anti-diagonal entries (n, D-1-n) by both (split_col).
constexpr int kMirD = 8;
// Level-5 (TMEM) lane maps, found by bank-conflict searches for the padded fan-out layout
// (tools/l5_layout_search.py): 128-bit shared-memory loads are served per 8-lane phase, so
// which parents share a phase decides the bank conflicts.  kL5VecMap: lane & 15 -> parent for
// the pivot / vector phase (conflict-free).  Nibble i = map(i).
constexpr uint64_t kL5VecMap = 0x79b0ec2568adf134ull;
__host__ __device__ __forceinline__ int l5_map(uint64_t map, int i) { return static_cast<int>((map >> (4 * i)) & 15); }

__host__ __device__ constexpr int mir_a_index(int i, int j) {  // index of (i,j) in A
    int n = 0;
    for (int a = 0; a < kMirD; ++a)
        for (int b = a; b < kMirD; ++b)
            if (a + b < kMirD - 1) {
                if (a == i && b == j) return n;
                ++n;
            }
    return -1;
}
__host__ __device__ constexpr int mir_a_row(int n) {
    for (int a = 0; a < kMirD; ++a)
        for (int b = a; b < kMirD; ++b)
            if (a + b < kMirD - 1 && n-- == 0) return a;
    return -1;
}
__host__ __device__ constexpr int mir_a_col(int n) {
    for (int a = 0; a < kMirD; ++a)
        for (int b = a; b < kMirD; ++b)
            if (a + b < kMirD - 1 && n-- == 0) return b;
    return -1;
}
// Split level-5 layout: a level-5 state row holds the 16 "A" entries (i + j < 7) in A order
// at columns U a, their 16 mirrors at 16 U + U a and the 4 anti-diagonal entries at 32 U + U n
// (U = words per entry; the row-0/1 entries the lane subtree loads first are then mostly
// consecutive A entries)
__host__ __device__ constexpr int split_col(int k, int U) {
    const int i = tri_row(kMirD, k), j = tri_col(kMirD, k);
    if (i + j == kMirD - 1) return 32 * U + U * i;
    return i + j < kMirD - 1 ? U * mir_a_index(i, j) : 16 * U + U * mir_a_index(kMirD - 1 - j, kMirD - 1 - i);
}
// TMEM column of entry k of a D-row lane state of word type T
template <class T, int D>
__host__ __device__ constexpr int tm_col(int k) {
    if constexpr (D == kMirD) return split_col(k, TmU<T>::U);
    else return TmU<T>::U * k;
}

// Rank-2 update of trailing entries [KB, KB+CNT) whose sources are in TMEM; the (i,j)
// of every entry is a template constant so u/w/Sn stay in registers.
template <class T, int M, int K, int END> struct LtUpd {
    __device__ __forceinline__ static void run(const uint32_t* rt, const T (&u)[M], const T (&w)[M],
                                               St<T, M / 2 - 1>& Sn) {
        if constexpr (K < END) {
            constexpr int D = M - 2;
            constexpr int i = tri_row(D, K), j = tri_col(D, K);
            Sn.e[K] = Arith<T>::rank2(from_u32<T>(rt), u[2 + i], u[2 + j], w[2 + i], w[2 + j]);
            LtUpd<T, M, K + 1, END>::run(rt + TmU<T>::U, u, w, Sn);
        }
    }
};
// Loads entries [K0, K0+N) of this lane's D-row TMEM state (issue only; tm_wait_ld
// before use).
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
// EPL entries in consecutive columns from entry K (one 16-column load / store)?
template <class T, int D, int K> __host__ __device__ constexpr bool tm_run16() {
    for (int q = 1; q < TmU<T>::EPL; ++q)
        if (tm_col<T, D>(K + q) != tm_col<T, D>(K) + TmU<T>::U * q) return false;
    return true;
}
template <class T, int D, int K, int N> struct TmLd {
    __device__ __forceinline__ static void run(uint32_t row, uint32_t* r) {
        if constexpr (N > 0) {
            constexpr int col = tm_col<T, D>(K), EPL = TmU<T>::EPL;
            // runs of EPL entries in consecutive columns (the natural scratch layout, the split
            // layout's A entries): one 16-column load
            if constexpr (N >= EPL && tm_run16<T, D, K>()) {
                tm_ld16(row + col, r);
                TmLd<T, D, K + EPL, N - EPL>::run(row, r + 16);
            } else {
                tm_ld_e<TmU<T>::U>(row + col, r);
                TmLd<T, D, K + 1, N - 1>::run(row, r + TmU<T>::U);
            }
        }
    }
};
template <class T, int D, int K0, int N>
__device__ __forceinline__ void tm_ld_entries(uint32_t row, uint32_t (&r)[TmU<T>::U * N]) {
    TmLd<T, D, K0, N>::run(row, r);
}
template <class T, int M, int KB, int CNT>
__device__ __forceinline__ void lt_wave(uint32_t row, const T (&u)[M], const T (&w)[M], St<T, M / 2 - 1>& Sn) {
    uint32_t rt[TmU<T>::U * CNT];
    tm_ld_entries<T, M, 2 * M - 1 + KB, CNT>(row, rt);
    tm_wait_ld();
    LtUpd<T, M, KB, KB + CNT>::run(rt, u, w, Sn);
}

// TMEM-streamed lane subtree: emits the 2^L - 1 extension terms of the L-mode node in
// this lane's TMEM row (its own term is emitted by the caller).  For L >= 4 the child
// states (L-1 modes) are not kept in registers: the include child is streamed entry
// by entry into the scratch columns scr (natural layout), the exclude child (the
// parent's trailing block) is copied there, and one copy of the (L-1)-mode code runs
// for both; the 3-mode level keeps its children (2 modes) in registers.
// entries K..K+Q-1 of the trailing update into 4Q words (compile-time (i,j))
template <class T, int M, int K, int Q> struct LtQuad {
    __device__ __forceinline__ static void run(const uint32_t* rt, const T (&u)[M], const T (&w)[M], uint32_t* r) {
        if constexpr (Q > 0) {
            constexpr int D = M - 2;
            constexpr int i = tri_row(D, K), j = tri_col(D, K);
            const T v = Arith<T>::rank2(from_u32<T>(rt), u[2 + i], u[2 + j], w[2 + i], w[2 + j]);
            to_u32(v, r);
            LtQuad<T, M, K + 1, Q - 1>::run(rt + TmU<T>::U, u, w, r + TmU<T>::U);
        }
    }
};
__device__ __forceinline__ void tm_st16p(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
template <class T, int M, int K, int END> struct LtUpdTm {
    __device__ __forceinline__ static void run(const uint32_t* rt, const T (&u)[M], const T (&w)[M], uint32_t dst) {
        if constexpr (K < END) {
            constexpr int D = M - 2;
            constexpr int i = tri_row(D, K), j = tri_col(D, K);
            constexpr int EPL = TmU<T>::EPL, U = TmU<T>::U;
            if constexpr (END - K >= EPL) {
                // EPL entries, one 16-column store (natural scratch layout)
                uint32_t r[16];
                LtQuad<T, M, K, EPL>::run(rt, u, w, r);
                tm_st16p(dst + tm_col<T, D>(K), r);
                LtUpdTm<T, M, K + EPL, END>::run(rt + 16, u, w, dst);
            } else {
                const T v = Arith<T>::rank2(from_u32<T>(rt), u[2 + i], u[2 + j], w[2 + i], w[2 + j]);
                uint32_t r[U];
                to_u32(v, r);
                tm_st_e<U>(dst + tm_col<T, D>(K), r);
                LtUpdTm<T, M, K + 1, END>::run(rt + U, u, w, dst);
            }
        }
    }
};
template <class T, int D, int K, int END> struct TmCopy {
    __device__ __forceinline__ static void run(const uint32_t* rt, uint32_t dst) {
        if constexpr (K < END) {
            constexpr int EPL = TmU<T>::EPL, U = TmU<T>::U;
            if constexpr (END - K >= EPL) {
                tm_st16p(dst + tm_col<T, D - 2>(K), rt);
                TmCopy<T, D, K + EPL, END>::run(rt + 16, dst);
            } else {
                tm_st_e<U>(dst + tm_col<T, D - 2>(K), rt);
                TmCopy<T, D, K + 1, END>::run(rt + U, dst);
            }
        }
    }
};
template <class T, int L, class AC, class E>
__device__ __forceinline__ void tmem_ext(uint32_t row, uint32_t scr, const T& t, bool neg, uint64_t mask, int nsel,
                                         AC& acc, E* err) {
    using A = Arith<T>;
    constexpr int M = 2 * L;
    constexpr int K01 = 2 * M - 1;  // entries of rows 0 and 1
    constexpr int NT = tri_sz(M - 2);
    constexpr int U = TmU<T>::U;
    const uint64_t bit = 1ull << (L - 1);
#pragma unroll 1
    for (int br = 0; br < 2; ++br) {
        T tn;
        if constexpr (L >= 4) {
            if (br == 0) {
                uint32_t r0[U * K01];
                tm_ld_entries<T, M, 0, K01>(row, r0);
                tm_wait_ld();
                T e0[K01];
#pragma unroll
                for (int k = 0; k < K01; ++k) e0[k] = from_u32<T>(r0 + U * k);
                const Piv<T> pv = piv_lt<T>(e0[0], e0[1], e0[M], t);
                if (pv.bad0 || pv.bad1) report_breakdown(err, mask | bit, 2 * nsel + (pv.bad0 ? 0 : 1));
                tn = pv.tn;
                T u[M], w[M];
#pragma unroll
                for (int j = 2; j < M; ++j) {
                    u[j] = A::mul(A::unb(e0[j]), pv.r1);
                    w[j] = A::mul(A::rank1s(e0[M + j - 1], pv.u1, u[j]), pv.r2);
                }
                constexpr int H = (NT + 2) / 3;
                {
                    uint32_t rt[U * H];
                    tm_ld_entries<T, M, K01, H>(row, rt);
                    tm_wait_ld();
                    LtUpdTm<T, M, 0, H>::run(rt, u, w, scr);
                }
                {
                    uint32_t rt[U * H];
                    tm_ld_entries<T, M, K01 + H, H>(row, rt);
                    tm_wait_ld();
                    LtUpdTm<T, M, H, 2 * H>::run(rt, u, w, scr);
                }
                {
                    uint32_t rt[U * (NT - 2 * H)];
                    tm_ld_entries<T, M, K01 + 2 * H, NT - 2 * H>(row, rt);
                    tm_wait_ld();
                    LtUpdTm<T, M, 2 * H, NT>::run(rt, u, w, scr);
                }
                acc.add(tn, !neg, nsel + 1);
            } else {
                constexpr int H = (NT + 1) / 2;
                {
                    uint32_t rt[U * H];
                    tm_ld_entries<T, M, K01, H>(row, rt);
                    tm_wait_ld();
                    TmCopy<T, M, 0, H>::run(rt, scr);
                }
                {
                    uint32_t rt[U * (NT - H)];
                    tm_ld_entries<T, M, K01 + H, NT - H>(row, rt);
                    tm_wait_ld();
                    TmCopy<T, M, H, NT>::run(rt, scr);
                }
                tn = t;
            }
            tm_wait_st();
            tmem_ext<T, L - 1, AC, E>(scr, scr, tn, br == 0 ? !neg : neg, br == 0 ? (mask | bit) : mask, nsel + (br == 0),
                                  acc, err);
        } else {
            St<T, L - 1> Sn;
            if (br == 0) {
                uint32_t r0[U * K01];
                tm_ld_entries<T, M, 0, K01>(row, r0);
                tm_wait_ld();
                T e0[K01];
#pragma unroll
                for (int k = 0; k < K01; ++k) e0[k] = from_u32<T>(r0 + U * k);
                const Piv<T> pv = piv_lt<T>(e0[0], e0[1], e0[M], t);
                if (pv.bad0 || pv.bad1) report_breakdown(err, mask | bit, 2 * nsel + (pv.bad0 ? 0 : 1));
                tn = pv.tn;
                T u[M], w[M];
#pragma unroll
                for (int j = 2; j < M; ++j) {
                    u[j] = A::mul(A::unb(e0[j]), pv.r1);
                    w[j] = A::mul(A::rank1s(e0[M + j - 1], pv.u1, u[j]), pv.r2);
                }
                lt_wave<T, M, 0, NT>(row, u, w, Sn);
                acc.add(tn, !neg, nsel + 1);
            } else {
                uint32_t rt[U * NT];
                tm_ld_entries<T, M, K01, NT>(row, rt);
                tm_wait_ld();
#pragma unroll
                for (int kk = 0; kk < NT; ++kk) Sn.e[kk] = from_u32<T>(rt + U * kk);
                tn = t;
            }
            SubReg<T, L - 1>::run(Sn, tn, br == 0 ? !neg : neg, br == 0 ? (mask | bit) : mask, nsel + (br == 0), acc,
                                  err);
        }
    }
}

// --------------------------------------------------------- subtree kernel ----
// Per-warp shared memory: the Q0-mode root (copy of the DFS leaf view), the
// include buffers of the fan-out levels, their t values, the pivot-row vectors and
// the DFS t values.  Per block: (i,j) tables of the fan-out child triangles.
template <class T> struct WarpSmem {
    static constexpr int L = Cfg<T>::L;
    static constexpr int Q0 = L + FAN;
    // Level-e include buffers: base lvl_off(e), child x at + x * buf_stride(e).  For the
    // TMEM (DD) layout the level-1 base is padded by 2 entries, the level-2 base by 1 and
    // the level-2 stride by 1 (5 entries per area): the 16 level-4 node states (level-5
    // parents, read lane-pair-wise by FanLevel<5>) then start on every 16-byte bank slot
    // mod 8 exactly twice and the 8 level-3 nodes on distinct slots, so those reads are
    // free of bank conflicts (found by exhaustive search over small paddings).
    // fp64 (8-byte words, level-5 states in shared memory): base pads, child stride adds, pair
    // strides and the fan-out lane maps of levels 1..5 from tools/f64_pairs_search.py, a bank
    // model of every fan-out access (pivot / vector loads, pair stores, item table / source /
    // pair loads and stores) and of the lane subtrees' level-5 reads (8-byte accesses served
    // per 16-lane phase, 16-byte per 8-lane phase): 1229 wavefronts per leaf against an ideal
    // of 1204 (the previous layout, tuned for the lane subtrees alone: 1681)
    static constexpr bool kF64Pad = sizeof(T) == sizeof(double) && !Cfg<T>::TMEM;
    // per level e = 1..5, 4 bits each from bit 4(e-1): base pads (13, 6, 1, 15, 0), stride adds
    // (6, 0, 3, 4, 3), pair strides m + (2, 2, 2, 1, 2) (16-byte units)
    static constexpr uint32_t kF64LvlPad = 0x0f16du, kF64StrideAdd = 0x34306u, kF64PairAdd = 0x21222u;
    static constexpr unsigned kF64Interleave = 0xeu;  // bit e-1: parent x = lane % E, else lane / G
    __host__ __device__ static constexpr int nib(uint32_t pack, int e) { return static_cast<int>((pack >> (4 * (e - 1))) & 15u); }
    __host__ __device__ static constexpr int lvl_pad(int e) {
        if constexpr (kF64Pad) return e >= 1 && e <= 5 ? nib(kF64LvlPad, e) : 0;
        return Cfg<T>::TMEM ? (e == 1 ? 2 : (e == 2 ? 1 : 0)) : 0;
    }
    __host__ __device__ static constexpr int buf_stride(int e) {
        if constexpr (kF64Pad) return tri_sz(2 * (Q0 - e)) + nib(kF64StrideAdd, e);
        return tri_sz(2 * (Q0 - e)) + (Cfg<T>::TMEM && e == 2 ? 1 : 0);
    }
    __host__ __device__ static constexpr int lvl_off(int e) {
        int o = tri_sz(2 * Q0);
        for (int x = 1; x < e; ++x) o += lvl_pad(x) + (1 << (x - 1)) * buf_stride(x);
        return e == 0 ? 0 : o + lvl_pad(e);
    }
    // with TMEM the last level's include states never touch shared memory
    static constexpr int kBufEntries = Cfg<T>::TMEM ? lvl_off(FAN) : lvl_off(FAN + 1);
    static constexpr int kTOff = kBufEntries;  // t of level buffers at 2^(e-1)-1+p, root t at 31
    // fp64 (unspecialised): the fan-out levels' pivot-row vectors are stored as (u_j, w_j)
    // pairs (one 16-byte load per index) and each parent's trailing items are run by its own
    // lane group with item tables indexed by the child entry alone (FanLevel)
    static constexpr bool kPairUw = sizeof(T) == sizeof(double) && !Cfg<T>::TMEM;
    // pair stride of a level-e parent (16-byte units, >= m = 2(Q0-e+1) pairs)
    __host__ __device__ static constexpr int uw_pair_stride(int e) { return 2 * (Q0 - e + 1) + nib(kF64PairAdd, e); }
    __host__ __device__ static constexpr int uw_need() {
        int mx = 4 * kMaxJobModes;  // DFS eliminations: 4q entries
        for (int e = 1; e <= FAN; ++e) {
            const int need = kPairUw ? (1 << (e - 1)) * 2 * uw_pair_stride(e)
                                     : (1 << (e - 1)) * (4 * (Q0 - e + 1) + 1);  // stride 2m+1 per parent
            if (need > mx) mx = need;
        }
        return mx;
    }
    static constexpr int kUwOff = kPairUw ? ((kTOff + 33) / 2) * 2 : kTOff + 32;  // pairs: 16-byte aligned
    static constexpr int kUwEntries = uw_need();
    static constexpr int kDfsT = kUwOff + kUwEntries;  // DFS slot t values (<= 32)
    // (warp-specialised: the DFS t values are producer-private, see kProdEntries)
    // (time-shared areas: the DFS t values of both warps)
    static constexpr int kEntries = kDfsT + (Cfg<T>::WS_MODE == 2 ? 0 : (Cfg<T>::TSHARE ? 64 : 32));
    // WS mode 2 producer-private: pivot-row vectors of the DFS and levels 1..3, DFS t
    // values of its two job contexts
    __host__ __device__ static constexpr int prod_uw() {
        int mx = 4 * kMaxJobModes;
        for (int e = 1; e <= 3; ++e) {
            const int need = (1 << (e - 1)) * (4 * (Q0 - e + 1) + 1);
            if (need > mx) mx = need;
        }
        return mx;
    }
    static constexpr int kProdUw = prod_uw();
    static constexpr int kProdEntries = kProdUw + 64;
    static constexpr size_t kWarpBytes = kEntries * sizeof(T);
    // Block-wide item tables of the fan-out trailing updates: level e has E*tn items
    // (it = x*tn + k: child x, entry k); word = src | ui << 12 | uj << 22 with src the
    // parent entry (index into the warp area; the smem layout is static, so this is a
    // constant per item), ui/uj the uw indices of u_i/u_j (w_i/w_j at +m).
    // Levels 1..kItemLevels use item tables; with TMEM the last level uses the (i,j)
    // table (ij_word) of its child triangle instead.
    static constexpr int kItemLevels = Cfg<T>::TMEM ? FAN - 1 : FAN;
    __host__ __device__ static constexpr int item_off(int e) {
        int o = 0;
        for (int x = 1; x < e; ++x) o += (kPairUw ? 1 : (1 << (x - 1))) * tri_sz(2 * (Q0 - x));
        return o;
    }
    static constexpr int kLastTabOff = item_off(kItemLevels + 1);
    // node offsets: node (e, c), e = 0..FAN, at kNodeOff + 2^e - 1 + c
    static constexpr int kNodeOff = kLastTabOff + (Cfg<T>::TMEM ? tri_sz(2 * (Q0 - FAN)) : 0);
    static constexpr int kTabEntries = kNodeOff + (2 << FAN) - 1;
    static constexpr size_t kTabBytes = ((kTabEntries * 4 + 15) / 16) * 16;
    static_assert(kBufEntries < 4096 && uw_need() <= 1024, "item word fields");
};

// Node (e, c) of the breadth-first fan-out rooted at the copied root (level 0): its
// state is a contiguous packed 2(Q0-e)-row triangle (an include buffer, or a view of
// an ancestor's trailing block for exclude chains) and its term factor t.
template <class T>
__device__ __forceinline__ int node_off(int e, int c) {
    constexpr int Q0 = WarpSmem<T>::Q0;
    if (c == 0) return tri_ix(2 * Q0, 2 * e, 2 * e);
    const int tz = __ffs(c) - 1;
    const int lvl = e - tz;
    const int p = (c >> tz) >> 1;
    const int dim = 2 * (Q0 - lvl);
    return WarpSmem<T>::lvl_off(lvl) + p * WarpSmem<T>::buf_stride(lvl) + tri_ix(dim, 2 * tz, 2 * tz);
}
__device__ __forceinline__ int node_tix(int e, int c) {
    if (c == 0) return 31;
    const int tz = __ffs(c) - 1;
    const int lvl = e - tz;
    return (1 << (lvl - 1)) - 1 + ((c >> tz) >> 1);
}
// node (e, c) from the per-block node table: word = node_off | node_tix << 16
struct NodeRef {
    int off, tix;
};
template <class T>
__device__ __forceinline__ NodeRef node_ref(const uint32_t* tabs, int e, int c) {
    const uint32_t w = tabs[WarpSmem<T>::kNodeOff + (1 << e) - 1 + c];
    return NodeRef{static_cast<int>(w & 0xffffu), static_cast<int>(w >> 16)};
}

// One breadth-first level: the E = 2^(e-1) include nodes of level e each eliminate
// the first mode of their parent (level e-1 node x) into level-e buffer x.  Lane
// (x, g) = (lane % E, lane / E) works on parent x throughout (pivots redundantly in
// registers, pivot-row vectors j = 2+g+sG, trailing entries k = g+sG, G = 32/E), so
// every source, table and destination address is a per-lane base plus a constant.
// Split level 5: threads x and x + 16 (x < 16) share parent kL5Split(x); their 128-bit
// loads of the parent's trailing block are served per 8-thread phase {0-7, 8-15, 16-23,
// 24-31}, so the parents of threads 0-7 (and of 8-15) must start on distinct 16-byte bank
// slots: the padded layout puts the 16 level-4 nodes on every slot exactly twice, and the map
// takes one of each slot for each half.
// conflict-free for the parent, anti-diagonal and pivot-row vector loads of the split
// chunks (144 wavefronts per leaf, the ideal; identity 224): tools/l5_split_search.py
constexpr uint64_t kL5Split = 0x3fc9a650e821b7d4ull;
// level-5 node in a consumer lane's TMEM row: lanes 0-15 the include children, 16-31 the
// exclude children of parents kL5Split(lane & 15)
__host__ __device__ __forceinline__ int l5_lane_node(int lane) {
    return 2 * l5_map(kL5Split, lane & 15) + (lane < 16 ? 1 : 0);
}
// 16x32bx2 stores: threads t and t + 16 write W columns each into TMEM lane t, the upper half
// SPLIT columns further (W = 4, 8 or 16 words)
template <int W, int SPLIT> __device__ __forceinline__ void tm_st_x2(uint32_t taddr, const uint32_t (&r)[W]) {
    if constexpr (W == 4) {
        asm volatile("tcgen05.st.sync.aligned.16x32bx2.x4.b32 [%0], %1, {%2, %3, %4, %5};\n" ::"r"(taddr), "n"(SPLIT),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]));
    } else if constexpr (W == 8) {
        asm volatile("tcgen05.st.sync.aligned.16x32bx2.x8.b32 [%0], %1, {%2, %3, %4, %5, %6, %7, %8, %9};\n" ::"r"(
                         taddr),
                     "n"(SPLIT), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    } else {
        static_assert(W == 16, "16x32bx2 store width");
        asm volatile(
            "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], %1, {%2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17};\n" ::"r"(taddr),
            "n"(SPLIT), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
            "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
}
// Chunk C (< 8): A entries 2C, 2C+1 (thread x) or their mirrors (thread x + 16) of the
// include child (computed) and of the exclude child (the parent's trailing block, raw):
// include rows at lanes 0-15, exclude rows at lanes 16-31, A at column 2UC, mirrors at +16U.
template <class T, int C> struct SplitChunk {
    __device__ __forceinline__ static void run(const T* Pt, const T (&u)[kMirD], const T (&w)[kMirD], int h,
                                               uint32_t tm_row) {
        if constexpr (C < 8) {
            using A = Arith<T>;
            constexpr int D = kMirD;
            constexpr int i0 = mir_a_row(2 * C), j0 = mir_a_col(2 * C);
            constexpr int i1 = mir_a_row(2 * C + 1), j1 = mir_a_col(2 * C + 1);
            constexpr int kA0 = cix<D>(i0, j0), kB0 = cix<D>(D - 1 - j0, D - 1 - i0);
            constexpr int kA1 = cix<D>(i1, j1), kB1 = cix<D>(D - 1 - j1, D - 1 - i1);
            const T in0 = Pt[h ? kB0 : kA0], in1 = Pt[h ? kB1 : kA1];
            const T v0 = A::rank2(in0, u[i0], u[j0], w[i0], w[j0]);
            const T v1 = A::rank2(in1, u[i1], u[j1], w[i1], w[j1]);
            constexpr int U = TmU<T>::U;
            uint32_t ri[2 * U], re[2 * U];
            to_u32(v0, ri);
            to_u32(v1, ri + U);
            to_u32(in0, re);
            to_u32(in1, re + U);
            tm_st_x2<2 * U, 16 * U>(tm_row + 2 * U * C, ri);
            tm_st_x2<2 * U, 16 * U>(tm_row + (16u << 16) + 2 * U * C, re);
            SplitChunk<T, C + 1>::run(Pt, u, w, h, tm_row);
        }
    }
};

#ifndef TOR_UB_P
#define TOR_UB_P 3  // producer fan-out levels (3 84.0, 4 84.2, 5 85.0, 6 84.3)
#endif
#ifndef TOR_UB
#define TOR_UB 4  // items per batch, consumer fan-out levels (n=32 DD: 4 84.1 ms, 5 85.0, 3 84.1)
#endif
#ifndef TOR_QD_UB
#define TOR_QD_UB 1
#endif
#ifndef TOR_F64_UB
#define TOR_F64_UB 5
#endif
// QD fan-out level trailing update: one out-of-line loop over this lane's items
// it = lane + 32 s (s < nit, it < ne), each s - u_i u_j - w_i w_j with the operands loaded
// from shared memory inside (one call per level instead of one per item)
__device__ __noinline__ void qd_items_ool(const qd* sm, const qd* uwv, const uint32_t* itb, qd* out, int nit, int ne,
                                          int m, int lane) {
#pragma unroll 1
    for (int s = 0; s < nit; ++s) {
        if (lane + 32 * s >= ne) break;
        const uint32_t w = itb[32 * s];
        const int src = static_cast<int>(w & 0xfffu);
        const int a = static_cast<int>((w >> 12) & 0x3ffu), b = static_cast<int>(w >> 22);
        out[32 * s] = qd_rank2_body<!kQdLazy>(sm[src], uwv[a], uwv[b], uwv[a + m], uwv[b + m]);
    }
}
template <class T, int E_LVL> struct FanLevel {
    static constexpr int Q0 = WarpSmem<T>::Q0;
    static constexpr int E = 1 << (E_LVL - 1);
    static constexpr int G = 32 / E;
    static constexpr int q = Q0 - E_LVL + 1;  // parent modes
    static constexpr int m = 2 * q;
    static constexpr int dn = m - 2;
    static constexpr int tn = tri_sz(dn);
    // fp64: lane (x, g) = (lane / G, lane % G) (the G lanes of parent x consecutive) or
    // (lane % E, lane / E) per level, whichever the bank search picked (WarpSmem).
    // Item k = g + sG of parent x: source Pt[k], destination out_x[k] (per-lane base + a
    // constant), (u, w) pairs of rows 2+i, 2+j at the byte offsets of table word k.
    // 10 instructions per item (4 loads, 3 integer, 2 DFMA, 1 store) instead of 17 for the
    // flat x-major item list with one decoded (src, ui, uj) word per item.
    template <class ErrSink>
    __device__ __forceinline__ static void run_pairs(double* sm, double* tvals, double* uwv, const uint32_t* tabs,
                                                     uint64_t leaf_mask, int leaf_sel, ErrSink* err) {
        using A = Arith<double>;
        using SM = WarpSmem<double>;
        const int lane = threadIdx.x & 31;
        constexpr bool kIl = (SM::kF64Interleave >> (E_LVL - 1)) & 1u;
        const int x = kIl ? lane % E : lane / G, g = kIl ? lane / E : lane % G;
        const double* P = sm + node_ref<double>(tabs, E_LVL - 1, x).off;
        const Piv<double> pv = pivot2<double>(P[0], P[1], P[m], tvals[node_ref<double>(tabs, E_LVL - 1, x).tix]);
        if (g == 0) {
            const uint64_t nm = leaf_mask | (static_cast<uint64_t>((x << 1) | 1) << (Q0 - E_LVL));
            if (pv.bad0 || pv.bad1) report_breakdown(err, nm, 2 * (leaf_sel + __popc(x)) + (pv.bad0 ? 0 : 1));
            tvals[E - 1 + x] = pv.tn;  // level e-1 t values live below index E-1: no hazard
        }
        constexpr int S2 = SM::uw_pair_stride(E_LVL);
        double2* uw2 = reinterpret_cast<double2*>(uwv) + x * S2;
        {
            constexpr int NVS = (m - 2 + G - 1) / G;
            double a[NVS], b[NVS];
#pragma unroll
            for (int s = 0; s < NVS; ++s) {
                const int j = 2 + g + s * G;  // reads past row end stay inside the warp area
                a[s] = P[j];
                b[s] = P[m - 1 + j];
            }
#pragma unroll
            for (int s = 0; s < NVS; ++s) A::vec(a[s], b[s], pv.r1, pv.u1, pv.r2, a[s], b[s]);
#pragma unroll
            for (int s = 0; s < NVS; ++s)
                if (g + s * G < m - 2) uw2[2 + g + s * G] = make_double2(a[s], b[s]);
        }
        __syncwarp();
        constexpr int NS = (tn + G - 1) / G;  // items per lane (the last one partial if tn % G)
        constexpr bool kPart = (tn % G) != 0;
        const char* uwb = reinterpret_cast<const char*>(uw2);
        const double* Pt = P + 2 * m - 1 + g;
        double* out = sm + SM::lvl_off(E_LVL) + x * SM::buf_stride(E_LVL) + g;
        const uint32_t* kt = tabs + SM::item_off(E_LVL) + g;
        const bool tail_ok = g < tn - (NS - 1) * G;
        auto batch = [&](int s0, auto cnt, auto last_partial) {
            constexpr int C = decltype(cnt)::value;
            constexpr bool LP = decltype(last_partial)::value;
            double sv[C];
            double2 pi[C], pj[C];
#pragma unroll
            for (int u = 0; u < C; ++u) {
                const uint32_t w = (!LP || u < C - 1 || tail_ok) ? kt[G * (s0 + u)] : 0u;
                sv[u] = Pt[G * (s0 + u)];
                pi[u] = *reinterpret_cast<const double2*>(uwb + (w & 0xffffu));
                pj[u] = *reinterpret_cast<const double2*>(uwb + (w >> 16));
            }
#pragma unroll
            for (int u = 0; u < C; ++u) sv[u] = A::rank2_item(sv[u], pi[u].x, pj[u].x, pi[u].y, pj[u].y);
#pragma unroll
            for (int u = 0; u < C; ++u)
                if (!LP || u < C - 1 || tail_ok) out[G * (s0 + u)] = sv[u];
        };
        constexpr int NFULL = NS - (kPart ? 1 : 0);
        constexpr int UB = TOR_F64_UB;
        constexpr int SMAIN = (NFULL / UB) * UB;
#pragma unroll 1
        for (int s0 = 0; s0 < SMAIN; s0 += UB) batch(s0, std::integral_constant<int, UB>{}, std::false_type{});
        constexpr int CT = NS - SMAIN;
        if constexpr (CT > 0) batch(SMAIN, std::integral_constant<int, CT>{}, std::integral_constant<bool, kPart>{});
        __syncwarp();
    }
    template <class ErrSink>
    __device__ __forceinline__ static void run(T* sm, T* tvals, T* uwv, const uint32_t* tabs, uint64_t leaf_mask,
                                               int leaf_sel, ErrSink* err, uint32_t tm_row) {
        if constexpr (WarpSmem<T>::kPairUw) {
            run_pairs(sm, tvals, uwv, tabs, leaf_mask, leaf_sel, err);
            return;
        }
        using A = Arith<T>;
        const int lane = threadIdx.x & 31;
        const int x = (Cfg<T>::TMEM && E_LVL == FAN) ? l5_map(kL5VecMap, lane & (E - 1)) : lane & (E - 1);
        const int g = lane / E;
        const NodeRef nr = node_ref<T>(tabs, E_LVL - 1, x);
        const T* P = sm + nr.off;
        // item-table words one batch ahead (the first batch's before the pivot chain): the
        // table read leaves each batch's load -> decode -> load -> update chain
        constexpr bool kItems = !(Cfg<T>::TMEM && E_LVL == FAN) && sizeof(T) != sizeof(qd);
        constexpr int UBQ = !Cfg<T>::WS ? TOR_F64_UB : (E_LVL < cons_first<T>() ? TOR_UB_P : TOR_UB);
        uint32_t wq[UBQ];
        if constexpr (kItems) {
#pragma unroll
            for (int u = 0; u < UBQ; ++u) wq[u] = tabs[WarpSmem<T>::item_off(E_LVL) + lane + 32 * u];
        }
        // (lanes l and l ^ E share parent x = l & (E - 1))
        const Piv<T> pv = pivot2_shared<T>(P[0], P[1], P[m], tvals[nr.tix], lane, E);
        if (g == 0) {
            const uint64_t nm = leaf_mask | (static_cast<uint64_t>((x << 1) | 1) << (Q0 - E_LVL));
            if (pv.bad0 || pv.bad1) report_breakdown(err, nm, 2 * (leaf_sel + __popc(x)) + (pv.bad0 ? 0 : 1));
            tvals[E - 1 + x] = pv.tn;  // level e-1 t values live below index E-1: no hazard
        }
        // pivot-row vectors u_j, w_j (j = 2..m-1) of parent x
        T* uwx = uwv + x * (2 * m + 1);  // odd stride: parents spread over the banks
        {
            constexpr int NVS = (m - 2 + G - 1) / G;
            T a[NVS], b[NVS];
#pragma unroll
            for (int s = 0; s < NVS; ++s) {
                const int j = 2 + g + s * G;  // reads past row end stay inside the warp area
                a[s] = P[j];
                b[s] = P[m - 1 + j];
            }
#pragma unroll
            for (int s = 0; s < NVS; ++s) {
                A::vec(a[s], b[s], pv.r1, pv.u1, pv.r2, a[s], b[s]);
            }
#pragma unroll
            for (int s = 0; s < NVS; ++s)
                if (g + s * G < m - 2) {
                    uwx[2 + g + s * G] = a[s];
                    uwx[m + 2 + g + s * G] = b[s];
                }
        }
        __syncwarp();
        if constexpr (Cfg<T>::TMEM && E_LVL == FAN) {
            // last level -> TMEM: threads x and x + 16 share parent kL5Split(x) and split
            // its include child's entries by the mirror (i,j) -> (7-j,7-i): thread x forms
            // the "A" entries (i+j < 7) with u, w in registers, thread x + 16 the mirrors
            // with the vectors held reversed -- the same register indices, so (i,j) are
            // compile-time for both.  16x32bx2 stores write both halves into ONE TMEM lane
            // (A at column 8C, mirrors at +64): lanes 0-15 receive the include children,
            // lanes 16-31 the exclude children (the parents' trailing blocks, loaded by the
            // same threads) -- no shuffles, no selects.  (Round 1's lane-pair mirror split
            // crossed results by shuffle + select: 84.1 vs 83.8 ms at n = 32.)
            static_assert(dn == kMirD && tn == 36 && E == 16, "mirror split layout");
            {
                const int xe = l5_map(kL5Split, lane & 15), h = lane >> 4;
                const T* Pt = sm + node_ref<T>(tabs, E_LVL - 1, xe).off + 2 * m - 1;
                const T* uwe = uwv + xe * (2 * m + 1);
                T u[dn], w[dn];
#pragma unroll
                for (int k = 0; k < dn; ++k) {
                    const int kk = 2 + (h ? dn - 1 - k : k);
                    u[k] = uwe[kk];
                    w[k] = uwe[m + kk];
                }
                SplitChunk<T, 0>::run(Pt, u, w, h, tm_row);
                constexpr int U = TmU<T>::U;
                uint32_t ri[4 * U], re[4 * U];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const T sv = Pt[cix<dn>(a, dn - 1 - a)];
                    to_u32(A::rank2(sv, u[dn - 1 - a], u[a], w[dn - 1 - a], w[a]), ri + U * a);
                    to_u32(sv, re + U * a);
                }
                // the anti-diagonal entries at column 32U (the upper half's duplicate at 36U lands
                // in the lane subtree's scratch columns, written only later)
                tm_st_x2<4 * U, 4 * U>(tm_row + 32 * U, ri);
                tm_st_x2<4 * U, 4 * U>(tm_row + (16u << 16) + 32 * U, re);
                tm_wait_st();
                __syncwarp();
                return;
            }
        }
        // trailing updates into the level-e buffers: item it = lane + 32 s (x-major)
        constexpr int NE = E * tn;
        constexpr int NIT = (NE + 31) / 32;
        constexpr int UB = sizeof(T) == sizeof(qd) ? TOR_QD_UB
                           : (!Cfg<T>::WS ? TOR_F64_UB : (E_LVL < cons_first<T>() ? TOR_UB_P : TOR_UB));  // items per batch
        const uint32_t* itb = tabs + WarpSmem<T>::item_off(E_LVL) + lane;
        T* out = sm + WarpSmem<T>::lvl_off(E_LVL) + lane;
        if constexpr (sizeof(T) == sizeof(qd)) {
            // QD: the item loop as one out-of-line call that loads its operands itself
            static_assert(WarpSmem<T>::buf_stride(E_LVL) == tn, "QD fan-out buffers are unpadded");
            qd_items_ool(reinterpret_cast<const qd*>(sm), reinterpret_cast<const qd*>(uwv), itb,
                         reinterpret_cast<qd*>(out), NIT, NE, m, lane);
            __syncwarp();
            return;
        }
        // batches of UB items every lane owns (no bounds checks), then one compile-time tail
        // batch: the remaining full items plus the partial last item (lanes < NE % 32)
        constexpr int NFULL = NE / 32, NREM = NE % 32;
        constexpr int SMAIN = (NFULL / UB) * UB;
        auto batch = [&](int s0, auto cnt, auto last_partial) {
            constexpr int C = decltype(cnt)::value;
            constexpr bool LP = decltype(last_partial)::value;
            T sv[C], ui[C], uj[C], wi[C], wj[C];
#pragma unroll
            for (int u = 0; u < C; ++u) {
                const bool ok = !LP || u < C - 1 || lane < NREM;
                const uint32_t w = ok ? wq[u] : 0u;
                const int src = static_cast<int>(w & 0xfffu);
                const int a = static_cast<int>((w >> 12) & 0x3ffu), b = static_cast<int>(w >> 22);
                sv[u] = sm[src];
                ui[u] = uwv[a];
                uj[u] = uwv[b];
                wi[u] = uwv[a + m];
                wj[u] = uwv[b + m];
            }
            if constexpr (C == UB && !LP) {  // a main batch: the next batch's words (reads past the
                                             // level's table stay inside shared memory, unused)
#pragma unroll
                for (int u = 0; u < UB; ++u) wq[u] = itb[32 * (s0 + UB + u)];
            }
#pragma unroll
            for (int u = 0; u < C; ++u) sv[u] = A::rank2_item(sv[u], ui[u], uj[u], wi[u], wj[u]);
#pragma unroll
            for (int u = 0; u < C; ++u) {
                const int s = s0 + u;
                if (!LP || u < C - 1 || lane < NREM) {
                    constexpr int kAdd = WarpSmem<T>::buf_stride(E_LVL) - tn;  // padded child stride
                    if constexpr (kAdd == 0) out[32 * s] = sv[u];
                    else out[32 * s + ((lane + 32 * s) / tn) * kAdd] = sv[u];
                }
            }
        };
#pragma unroll 1
        for (int s0 = 0; s0 < SMAIN; s0 += UB) batch(s0, std::integral_constant<int, UB>{}, std::false_type{});
        constexpr int CT = NFULL - SMAIN + (NREM ? 1 : 0);
        if constexpr (CT > 0) batch(SMAIN, std::integral_constant<int, CT>{}, std::integral_constant<bool, NREM != 0>{});
        __syncwarp();
    }
};


// kScaled: the input was scaled by 2^-tsc (Acc)
template <class T, bool kScaled>
__global__ void __launch_bounds__(32 * Cfg<T>::WPB, Cfg<T>::MINB)
    subtree_kernel(const Job<T>* jobs, uint64_t njobs, int nmodes, int rjob, T* scratch, size_t scratch_stride,
                   double* partials, unsigned long long* err, unsigned long long* job_counter, int tsc) {
    using SM = WarpSmem<T>;
    constexpr int L = Cfg<T>::L;
    constexpr int Q0 = SM::Q0;
    constexpr int WPB = Cfg<T>::WPB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* tabs = reinterpret_cast<uint32_t*>(smem_raw);
    // block-wide item tables of the fan-out levels (see WarpSmem)
    for (int e = 1; e <= SM::kItemLevels; ++e) {
        const int m = 2 * (Q0 - e + 1), D = m - 2, tn = tri_sz(D);
        if constexpr (SM::kPairUw) {
            // child entry k = (i, j): byte offsets of the pairs 2+i, 2+j in the parent's pair array
            for (int k = threadIdx.x; k < tn; k += blockDim.x) {
                int i = 0, r = k;
                while (r >= D - i) {
                    r -= D - i;
                    ++i;
                }
                tabs[SM::item_off(e) + k] = static_cast<uint32_t>(16 * (2 + i)) |
                                            (static_cast<uint32_t>(16 * (2 + i + r)) << 16);
            }
            continue;
        }
        for (int it = threadIdx.x; it < (tn << (e - 1)); it += blockDim.x) {
            const int x = it / tn;
            int i = 0, r = it - x * tn;
            while (r >= D - i) {
                r -= D - i;
                ++i;
            }
            const int src = node_off<T>(e - 1, x) + 2 * m - 1 + (it - x * tn);
            const int ui = x * (2 * m + 1) + 2 + i, uj = x * (2 * m + 1) + 2 + i + r;
            tabs[SM::item_off(e) + it] = static_cast<uint32_t>(src) | (static_cast<uint32_t>(ui) << 12) |
                                         (static_cast<uint32_t>(uj) << 22);
        }
    }
    for (int e = 0; e <= FAN; ++e)
        for (int c = threadIdx.x; c < (1 << e); c += blockDim.x) tabs[SM::kNodeOff + (1 << e) - 1 + c] =
                static_cast<uint32_t>(node_off<T>(e, c)) | (static_cast<uint32_t>(node_tix(e, c)) << 16);
    if constexpr (Cfg<T>::TMEM) {
        const int D = 2 * (Q0 - FAN);
        for (int k = threadIdx.x; k < tri_sz(D); k += blockDim.x) {
            int i = 0, r = k;
            while (r >= D - i) {
                r -= D - i;
                ++i;
            }
            tabs[SM::kLastTabOff + k] = ij_word(i, i + r);
        }
    }
    __shared__ uint32_t tmem_base;
    // time-shared areas: whose turn it is (0 / 1 = warp w < 4 / w >= 4) and who has finished
    __shared__ volatile int ts_turn[4], ts_done[8];
    __shared__ unsigned long long ts_ls[2];
    if (threadIdx.x < 2) ts_ls[threadIdx.x] = 0ull;
    if constexpr (Cfg<T>::TSHARE) {
        if (threadIdx.x < 4) ts_turn[threadIdx.x] = 0;
        if (threadIdx.x < 8) ts_done[threadIdx.x] = 0;
    }
    constexpr bool kUseTmem = Cfg<T>::TMEM || Cfg<T>::TSHARE;
    uint32_t tm_row = 0;
    if constexpr (kUseTmem) {
        // warp w uses TMEM lanes 32(w%4).. (its lane quadrant) and columns 256(w/4)..
        static_assert(Cfg<T>::WPB == 4 || Cfg<T>::WPB == 8 || Cfg<T>::WPB == 12, "TMEM lane handoff: 4, 8, 12 warps");
        constexpr uint32_t kCols = Cfg<T>::WPB >= 8 ? 512 : 256;
        if ((threadIdx.x >> 5) == 0) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base));
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(dst), "r"(kCols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        tm_row = tmem_base + (static_cast<uint32_t>(32 * ((threadIdx.x >> 5) & 3)) << 16) + 256u * (threadIdx.x >> 7);
    } else {
        __syncthreads();
    }
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int D = rjob - Q0;
    // DFS slot s (state after the include at depth s-1, 2(rjob-s) rows) starts at entry
    // sum_{x=1}^{s-1} tri(2(rjob-x)); lane s keeps that offset
    int slot_off_l = 0;
    for (int x = 1; x < lane && x <= D; ++x) slot_off_l += tri_sz(2 * (rjob - x));
    // Warp areas.  Unspecialised: warp w owns area w.  Warp-specialised: the pair
    // (producer p, consumer p+4) owns areas 2p and 2p+1; their fan-out buffers and t
    // values alternate between leaves (slot = leaf parity), the pivot-row vectors of
    // area 2p are the producer's, those of area 2p+1 the consumer's (level FAN).
    // WS mode 2: areas 0..7 belong to the consumers (producer p fills areas p, p+4);
    // producer p's private pivot-row vectors and DFS t values follow the areas.
    const int pw = Cfg<T>::WS ? (wib & 3) : wib;
    const int ppb = Cfg<T>::WS ? 4 : WPB;  // producers per block
    auto area = [&](int a) { return reinterpret_cast<T*>(smem_raw + SM::kTabBytes + a * SM::kWarpBytes); };
    T* sm = area(Cfg<T>::WS_MODE == 2 ? pw : (Cfg<T>::WS ? 2 * pw : (Cfg<T>::TSHARE ? (wib & 3) : pw)));
    T* tvals = sm + SM::kTOff;
    T* uwv = Cfg<T>::WS_MODE == 2 ? area(8) + pw * SM::kProdEntries : sm + SM::kUwOff;
    T* dfs_t = Cfg<T>::WS_MODE == 2 ? uwv + SM::kProdUw : sm + SM::kDfsT + (Cfg<T>::TSHARE ? 32 * (wib >> 2) : 0);
    T* slots = scratch + static_cast<size_t>(blockIdx.x * ppb + pw) * scratch_stride;

    // DFS step + root + fan-out of one leaf of job J into the fan area fsm (buffers +
    // t values): all FAN levels, or (warp-specialised) levels 1..FAN-1 -- the level-FAN
    // states in shared memory, or in TMEM at tm_slot for the TMEM types
    unsigned long long* perr = err;
    // time-shared areas: lock-step rounds of the warp's group (see the leaf loop)
    unsigned long long ts_k = 0;
    auto ts_sync = [&](unsigned long long target) {
        if (lane == 0) atomicAdd(&ts_ls[wib >> 2], 1ull);
        __syncwarp();
        while (*reinterpret_cast<volatile unsigned long long*>(&ts_ls[wib >> 2]) < target) __nanosleep(20);
    };
    auto produce_leaf = [&](const Job<T>& J, uint64_t leaf, uint32_t tm_slot, T* fsm, T* dfs_t, T* slots) {
        T* ftv = fsm + SM::kTOff;
        if (leaf > 0) {
            // flip exclude->include at depth kd (lowest set bit of leaf)
            const int b = __ffsll(static_cast<long long>(leaf)) - 1;
            const int kd = D - 1 - b;
            const uint64_t above = leaf >> (b + 1);
            const T* src;
            T st;
            if (above == 0) {
                const int sk = 2 * (J.skip + kd);
                src = J.base + tri_ix(J.dim, sk, sk);
                st = J.t;
            } else {
                const int tz = __ffsll(static_cast<long long>(above)) - 1;
                const int s = kd - tz;  // slot index (depth after that include)
                src = slots + __shfl_sync(0xffffffffu, slot_off_l, s) + tri_ix(2 * (rjob - s), 2 * tz, 2 * tz);
                st = dfs_t[s];
            }
            const int doff = __shfl_sync(0xffffffffu, slot_off_l, kd + 1);
            const uint64_t lmask = J.mask | ((above << 1 | 1ull) << (rjob - kd - 1));
            const int lsel = J.nsel + __popcll(above);
            // the new slot kd+1 is re-read by later leaves only when b >= 1; its
            // trailing Q0 modes are this leaf's root either way
            dfs_elim<T, Q0>(src, rjob - kd, slots + doff, b >= 1, fsm, st, dfs_t + kd + 1, uwv,
                            g_ijtab + ijtab_off(rjob - kd - 1), lmask, lsel, err);
            if (lane == 0) ftv[31] = dfs_t[kd + 1];
            __syncwarp();
        }
        if (leaf == 0) {
            // first leaf: the root is the job state's trailing Q0 modes (HBM), a
            // contiguous packed triangle
            const int sk = 2 * (J.skip + D);
            const T* lb = J.base + tri_ix(J.dim, sk, sk);
            constexpr int RT = tri_sz(2 * Q0);
            constexpr int RI = (RT + 31) / 32;
            T rv[RI];
#pragma unroll
            for (int s = 0; s < RI; ++s) {
                const int k0 = lane + 32 * s;
                rv[s] = lb[k0 < RT ? k0 : RT - 1];
            }
#pragma unroll
            for (int s = 0; s < RI; ++s)
                if (lane + 32 * s < RT) fsm[lane + 32 * s] = rv[s];
            if (lane == 0) ftv[31] = J.t;
        }
        __syncwarp();
        const uint64_t leaf_mask = J.mask | (leaf << Q0);
        const int leaf_sel = J.nsel + __popcll(leaf);
        // fan-out levels 1 .. cons_first - 1 (all of them when unspecialised)
        constexpr int CF = Cfg<T>::WS ? cons_first<T>() : FAN + 1;
        if constexpr (CF > 1) FanLevel<T, 1>::run(fsm, ftv, uwv, tabs, leaf_mask, leaf_sel, perr, tm_slot);
        if constexpr (CF > 2) FanLevel<T, 2>::run(fsm, ftv, uwv, tabs, leaf_mask, leaf_sel, perr, tm_slot);
        if constexpr (CF > 3) FanLevel<T, 3>::run(fsm, ftv, uwv, tabs, leaf_mask, leaf_sel, perr, tm_slot);
        if constexpr (CF > 4) FanLevel<T, 4>::run(fsm, ftv, uwv, tabs, leaf_mask, leaf_sel, perr, tm_slot);
        if constexpr (CF > 5) FanLevel<T, 5>::run(fsm, ftv, uwv, tabs, leaf_mask, leaf_sel, perr, tm_slot);
    };
    using AccT = Acc<T, kScaled>;
    auto write_partial = [&](AccT& acc, unsigned long long job) {
        warp_fold(acc);
        if (lane == 0) {
            double w[4];
            acc.words(w);
            double* o = partials + job * 5;
            o[0] = w[0];
            o[1] = w[1];
            o[2] = w[2];
            o[3] = w[3];
            o[4] = acc.abs_sum;
        }
        __syncwarp();
    };

    if constexpr (Cfg<T>::WS_MODE == 2) {
        // ---- warp-specialised, 4 producers + 8 consumers.  Producer p keeps two job
        // contexts s = 0, 1; leaf after leaf it alternates between them, running the DFS
        // and fan-out levels 1..3 of context s into consumer (p + 4s)'s area.  Consumer c
        // runs levels 4 and 5 (TMEM, its lane quadrant c % 4, columns 256 (c / 4)) and
        // the lane subtrees, accumulating whole jobs (same per-job arithmetic and order
        // as the unspecialised kernel).  Areas are handed over by mbarriers: full[c]
        // (producer -> consumer), empty[c] (consumer -> producer, arrived as soon as the
        // consumer no longer reads the producer's part of the area).
        struct WsMeta {
            unsigned long long mask;
            unsigned long long job;
            int sel, flags;  // 1: last leaf of the job, 2: no more leaves
        };
        __shared__ WsMeta meta[8];
        __shared__ __align__(8) unsigned long long mbar[16];  // full[0..7], empty[8..15]
        if (threadIdx.x < 16) {
            const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[threadIdx.x]));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(32) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        __syncthreads();
        auto mb_arrive = [&](int i) {
            const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[i]));
            asm volatile("{.reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0];}\n" ::"r"(a) : "memory");
        };
        auto mb_wait = [&](int i, uint32_t parity) {
            const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[i]));
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p;}\n"
                    : "=r"(ok)
                    : "r"(a), "r"(parity), "r"(static_cast<uint32_t>(TOR_MB_HINT))
                    : "memory");
        };
        if (wib < 4) {
            const int p = wib;
            Job<T> J[2];
            unsigned long long jid[2];
            uint64_t leaf[2] = {0, 0};
            bool act[2];
            uint32_t uses[2] = {0, 0};
            auto fetch = [&](int s) {
                unsigned long long j = 0;
                if (lane == 0) j = atomicAdd(job_counter, 1ull);
                j = __shfl_sync(0xffffffffu, j, 0);
                act[s] = j < njobs;
                jid[s] = j;
                if (act[s]) J[s] = jobs[j];
                leaf[s] = 0;
            };
            fetch(0);
            fetch(1);
            while (act[0] || act[1]) {
#pragma unroll 1
                for (int s = 0; s < 2; ++s) {
                    if (!act[s]) continue;
                    const int c = p + 4 * s;
                    mb_wait(8 + c, (uses[s] & 1) ^ 1);
                    T* cslots = scratch + (static_cast<size_t>(blockIdx.x * 4 + p) * 2 + s) * scratch_stride;
                    produce_leaf(J[s], leaf[s], 0u, area(c), dfs_t + 32 * s, cslots);
                    if (lane == 0) {
                        meta[c].mask = J[s].mask | (leaf[s] << Q0);
                        meta[c].job = jid[s];
                        meta[c].sel = J[s].nsel + __popcll(leaf[s]);
                        meta[c].flags = leaf[s] + 1 == (1ull << D) ? 1 : 0;
                    }
                    __syncwarp();
                    mb_arrive(c);
                    ++uses[s];
                    if (++leaf[s] == (1ull << D)) fetch(s);
                }
            }
#pragma unroll 1
            for (int s = 0; s < 2; ++s) {
                const int c = p + 4 * s;
                mb_wait(8 + c, (uses[s] & 1) ^ 1);
                if (lane == 0) meta[c].flags = 2;
                __syncwarp();
                mb_arrive(c);
            }
        } else {
            const int c = wib - 4;
            const uint32_t crow = tmem_base + ((32u * (c & 3)) << 16) + 256u * (c >> 2);
            T* csm = area(c);
            T* ctv = csm + SM::kTOff;
            T* cuw = csm + SM::kUwOff;
            AccT acc;
            acc.sc = tsc;
            LocalErr lerr;
            LocalErr* cerr = &lerr;
            for (uint32_t k = 0;; ++k) {
                mb_wait(c, k & 1);
                const unsigned long long leaf_mask = meta[c].mask;
                const unsigned long long job = meta[c].job;
                const int leaf_sel = meta[c].sel, flags = meta[c].flags;
                if (flags & 2) break;
                if constexpr (cons_first<T>() <= 2) FanLevel<T, 2>::run(csm, ctv, cuw, tabs, leaf_mask, leaf_sel, cerr, crow);
                if constexpr (cons_first<T>() <= 3) FanLevel<T, 3>::run(csm, ctv, cuw, tabs, leaf_mask, leaf_sel, cerr, crow);
                if constexpr (cons_first<T>() <= 4) FanLevel<T, 4>::run(csm, ctv, cuw, tabs, leaf_mask, leaf_sel, cerr, crow);
                FanLevel<T, FAN>::run(csm, ctv, cuw, tabs, leaf_mask, leaf_sel, cerr, crow);
                const int node = l5_lane_node(lane);  // the level-5 node in this lane's TMEM row
                const T vt = ctv[node_ref<T>(tabs, FAN, node).tix];
                __syncwarp();
                mb_arrive(8 + c);  // the producer may refill root..L3 and t values 0..6, 31
                const uint64_t lmask = leaf_mask | (static_cast<uint64_t>(node) << L);
                const int lsel = leaf_sel + __popc(node);
                const bool nodeneg = ((nmodes - lsel) & 1) != 0;  // term sign (-1)^(n - |Z|)
                acc.add(vt, nodeneg, lsel);
                tmem_ext<T, L, AccT>(crow, crow + TmU<T>::U * tri_sz(2 * L), vt, nodeneg, lmask, lsel, acc, cerr);
                acc.flush();
                if (flags & 1) {
                    write_partial(acc, job);
                    acc = AccT();
                    acc.sc = tsc;
                }
            }
            lerr.flush(err);
        }
    } else {
        for (;;) {
            unsigned long long job = 0;
            if (lane == 0) job = atomicAdd(job_counter, 1ull);
            job = __shfl_sync(0xffffffffu, job, 0);
            if (job >= njobs) break;
            const Job<T> J = jobs[job];
            AccT acc;
            acc.sc = tsc;
            for (uint64_t leaf = 0; leaf < (1ull << D); ++leaf) {
                if constexpr (Cfg<T>::TSHARE) {
                    // wait for the area: my turn, or the partner warp has no more leaves.  Every
                    // lane polls (one broadcast load per trip, a warp-uniform exit): a single polling
                    // lane left the warp split in two groups that each ran the whole leaf
                    while (ts_turn[wib & 3] != (wib >> 2) && !ts_done[wib ^ 4]) __nanosleep(64);
                    __syncwarp();
                    __threadfence_block();
                    // The four holders of a phase start their fan-out together: warps that run the
                    // same code at the same time share its instruction fetches (n = 32: 1285 -> 1176
                    // ms, n = 28: 72.9 -> 71.0; a desynchronised pool of areas ran at half the speed;
                    // further meetings per leaf gain nothing).  Arrival counter per group; a finished
                    // warp credits all later rounds.
                    ++ts_k;
                    ts_sync(4ull * ts_k);
                }
                produce_leaf(J, leaf, tm_row, sm, dfs_t, slots);
                // lanes: node (FAN, c); TMEM rows hold the nodes of the level-5 lane map
                const uint64_t leaf_mask = J.mask | (leaf << Q0);
                const int leaf_sel = J.nsel + __popcll(leaf);
                const int c = lane;
                const NodeRef nr = node_ref<T>(tabs, FAN, c);
                const T vt = tvals[nr.tix];
                const uint64_t lmask = leaf_mask | (static_cast<uint64_t>(c) << L);
                const int lsel = leaf_sel + __popc(c);
                const bool nodeneg = ((nmodes - lsel) & 1) != 0;  // term sign (-1)^(n - |Z|)
                if constexpr (Cfg<T>::TSHARE) {
                    // the lane's node state (a contiguous packed 2L-row triangle) -> its TMEM row,
                    // then the area goes to the partner warp
                    constexpr int U = TmU<T>::U;
#pragma unroll
                    for (int k = 0; k < tri_sz(2 * L); ++k) {
                        uint32_t r[U];
                        to_u32(sm[nr.off + k], r);
                        tm_st_e<U>(tm_row + static_cast<uint32_t>(U * k), r);
                    }
                    tm_wait_st();
                    __syncwarp();
                    __threadfence_block();
                    ts_turn[wib & 3] = (wib >> 2) ^ 1;  // (every lane stores the same value: no divergence)
                    lane_tree_v<T, L, AccT>(TmemView<T, 2 * L>{tm_row}, vt, nodeneg, lmask, lsel, acc, err);
                } else {
                    lane_tree<T, L, AccT>(sm + nr.off, 2 * L, 0, vt, nodeneg, lmask, lsel, acc, err);
                }
                acc.flush();
                __syncwarp();
            }
            write_partial(acc, job);
        }
        if constexpr (Cfg<T>::TSHARE) {
            __syncwarp();
            __threadfence_block();
            if (lane == 0) atomicAdd(&ts_ls[wib >> 2], 1ull << 40);
            __syncwarp();
            ts_done[wib] = 1;
        }
    }
    if constexpr (kUseTmem) {
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        if ((threadIdx.x >> 5) == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                         "r"(Cfg<T>::WPB >= 8 ? 512 : 256)
                         : "memory");
    }
}

// ----------------------------------------------------------- small jobs ----
// Jobs whose state has fewer than Q0 modes (small n, deep slices): one thread per
// job enumerates all 2^r subsets W of the job modes with a direct Cholesky of the
// gathered 2|W| x 2|W| Schur-complement submatrix.
template <class T, int RMAX>
__global__ void small_job_kernel(const Job<T>* jobs, uint64_t njobs, int nmodes, int rjob, double* partials,
                                 unsigned long long* err, int tsc) {
    using A = Arith<T>;
    const uint64_t jid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (jid >= njobs) return;
    const Job<T> J = jobs[jid];
    Acc<T, true> acc;  // runtime scale (small jobs are off the hot path)
    acc.sc = tsc;
    T M[tri_sz(2 * RMAX)];
    int sel[RMAX];
    for (uint64_t w = 0; w < (1ull << rjob); ++w) {
        int z = 0;
        for (int m = 0; m < rjob; ++m)
            if ((w >> (rjob - 1 - m)) & 1) sel[z++] = m;
        const int d = 2 * z;
        for (int a = 0; a < d; ++a)
            for (int b = a; b < d; ++b) {
                const int ra = 2 * (J.skip + sel[a >> 1]) + (a & 1);
                const int rb = 2 * (J.skip + sel[b >> 1]) + (b & 1);
                M[tri_ix(d, a, b)] = A::unb(J.base[tri_ix(J.dim, ra, rb)]);
            }
        T t = J.t;
        const uint64_t mask = J.mask | w;
        for (int k = 0; k < d; ++k) {
            const T p = A::norm(M[tri_ix(d, k, k)]);
            if (nonpositive(A::hi(p))) report_breakdown(err, mask, 2 * J.nsel + k);
            const T r = A::rsqrt(p);
            t = A::mul(t, r);
            for (int j = k + 1; j < d; ++j) M[tri_ix(d, k, j)] = A::mul(M[tri_ix(d, k, j)], r);
            for (int i = k + 1; i < d; ++i)
                for (int j = i; j < d; ++j)
                    M[tri_ix(d, i, j)] = A::rank1(M[tri_ix(d, i, j)], M[tri_ix(d, k, i)], M[tri_ix(d, k, j)]);
        }
        const bool neg = ((nmodes - J.nsel - z) & 1) != 0;
        acc.add(t, neg, J.nsel + z);
        acc.flush();
    }
    double wds[4];
    acc.words(wds);
    double* o = partials + jid * 5;
    for (int i = 0; i < 4; ++i) o[i] = wds[i];
    o[4] = acc.abs_sum;
}

// ------------------------------------------------------------- reduction ----
template <class T> __host__ __device__ inline void merge_words(double* a, const double* b) {
    if constexpr (sizeof(T) == sizeof(qd)) {
        const qd x{{a[0], a[1], a[2], a[3]}};
        const qd y{{b[0], b[1], b[2], b[3]}};
        const qd r = qd_add(x, y);
        for (int i = 0; i < 4; ++i) a[i] = r.x[i];
    } else {
        const dd r = dd_add(dd{a[0], a[1]}, dd{b[0], b[1]});
        a[0] = r.hi;
        a[1] = r.lo;
        a[2] = 0.0;
        a[3] = 0.0;
    }
    a[4] += b[4];
}

// Fixed binary tree over an instance's `per` consecutive job partials (5 doubles
// each): at stride s = 1, 2, 4, ... partial i (i = 0 mod 2s) absorbs partial i + s
// (when i + s < per); the result lands in partial 0.  One pass folds, per block,
// kFoldB consecutive elements of the level-S array (element k = partial k*S) -- an
// aligned subtree of the same tree -- into its first element; passes at S = 1,
// kFoldB, kFoldB^2, ... reproduce the whole tree exactly (bit-identical to a single
// sequential fold, and to fold_words on the host).
constexpr int kFoldB = 512;
// G (a power of two <= kFoldB): groups of G elements fold separately, stopping the tree at
// subtrees of G*S partials (the per-class partials of WorkRange::class_partials).
template <class T>
__global__ void __launch_bounds__(kFoldB / 2) fold_pass_kernel(double* partials, uint64_t per, uint64_t S, int inst0,
                                                               int G) {
    __shared__ double sh[kFoldB * 5];
    double* p = partials + (inst0 + static_cast<uint64_t>(blockIdx.y)) * per * 5;
    const uint64_t cnt = (per + S - 1) / S;
    const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * kFoldB;
    for (int x = threadIdx.x; x < kFoldB * 5; x += blockDim.x) {
        const uint64_t k = k0 + x / 5;
        sh[x] = k < cnt ? p[(k * S) * 5 + x % 5] : 0.0;
    }
    __syncthreads();
    for (int s = 1; s < G; s <<= 1) {
        const int i = threadIdx.x * 2 * s;
        if (i < kFoldB && k0 + i + s < cnt) merge_words<T>(sh + i * 5, sh + (i + s) * 5);
        __syncthreads();
    }
    for (int x = threadIdx.x; x < (kFoldB / G) * 5; x += blockDim.x) {
        const uint64_t k = k0 + static_cast<uint64_t>(x / 5) * G;
        if (k < cnt) p[(k * S) * 5 + x % 5] = sh[(x / 5) * G * 5 + x % 5];
    }
}

// Contiguous uploaded inputs (ninst x words doubles) into the pool's per-instance level-0
// buffers (stride `stride` doubles).  A strided copy-engine transfer runs row by row.
__global__ void scatter_inputs_kernel(const double* in, uint64_t words, int ninst, uint64_t stride, double* pool) {
    const uint64_t total = words * ninst;
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        pool[(k / words) * stride + k % words] = in[k];
}

// Result words of every instance (partial 0 of its job range) and the breakdown word into
// one contiguous buffer: a single device->host copy instead of one row per instance.
__global__ void gather_results_kernel(const double* partials, uint64_t per, int ninst,
                                      const unsigned long long* err, double* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < ninst * 5) out[k] = partials[static_cast<uint64_t>(k / 5) * per * 5 + k % 5];
    if (k == 0) reinterpret_cast<unsigned long long*>(out)[ninst * 5] = *err;
}

// ------------------------------------------------------------ host side ----
#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            err = std::string(#x) + ": " + cudaGetErrorString(e_);                    \
            return static_cast<int>(e_);                                              \
        }                                                                             \
    } while (0)

// Process-wide cache of device allocations: plans are created per call (the C ABI
// is stateless), and cudaMalloc/cudaFree of the tens of MB of prefix pools and DFS
// scratch would otherwise cost milliseconds per call.  Blocks are reused when their
// capacity is within 2x of the request; tor_release_device_cache() frees them.
struct DevPool {
    static constexpr size_t kMaxPooled = size_t(8) << 30;  // per device
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks[64];
    size_t pooled[64] = {};
    static DevPool& get() {
        static DevPool pool;
        return pool;
    }
};
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    int dev = -1;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    cudaError_t alloc(size_t bytes, int device) {
        bytes = std::max<size_t>(bytes, 256);
        if (device >= 0 && device < 64) {
            DevPool& pl = DevPool::get();
            std::lock_guard<std::mutex> lk(pl.mu);
            auto& fb = pl.free_blocks[device];
            auto it = fb.lower_bound(bytes);
            if (it != fb.end() && it->first <= 2 * bytes) {
                p = it->second;
                cap = it->first;
                dev = device;
                pl.pooled[device] -= cap;
                fb.erase(it);
                return cudaSuccess;
            }
        }
        const cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) {
            cap = bytes;
            dev = device;
        } else {
            p = nullptr;
        }
        return e;
    }
    ~DevBuf() {
        if (!p) return;
        if (dev >= 0 && dev < 64) {
            DevPool& pl = DevPool::get();
            std::lock_guard<std::mutex> lk(pl.mu);
            if (pl.pooled[dev] + cap <= DevPool::kMaxPooled) {
                pl.free_blocks[dev].emplace(cap, p);
                pl.pooled[dev] += cap;
                return;
            }
        }
        cudaFree(p);
    }
};

// (i,j) tables of the DFS eliminations, uploaded once per device
int ensure_ijtab(int device, std::string& err) {
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (device >= 0 && device < 64 && done[device]) return 0;
    std::vector<uint32_t> h(kIjTabEntries);
    for (int a = 1; a < kMaxJobModes; ++a) {
        const int D = 2 * a;
        int k = ijtab_off(a);
        for (int i = 0; i < D; ++i)
            for (int j = i; j < D; ++j) h[k++] = ij_word(i, j);
    }
    CK(cudaMemcpyToSymbol(g_ijtab, h.data(), sizeof(uint32_t) * h.size()));
    if (device >= 0 && device < 64) done[device] = true;
    return 0;
}

// A prepared evaluation: geometry chosen, device buffers allocated, the exact R of
// every instance resident in HBM.  execute() runs the whole device pipeline
// (prefix levels -> jobs -> subtree kernel -> fixed-order fold) and reads back
// 5 doubles per instance; it can be called repeatedly (inputs stay resident).
template <class T>
class PlanImpl final : public Plan {
  public:
    int init(int device, const std::vector<PreparedInput>& inputs, const WorkRange& range, std::string& err) {
        constexpr int K = Arith<T>::K;
        if (const int st = init_geometry(device, inputs[0].n, static_cast<int>(inputs.size()), range, err)) return st;
        // resident inputs: the exact R of every instance, one strided copy for the batch
        const size_t rt = static_cast<size_t>(tri_sz(2 * n_)) * K;
        std::vector<double> host(rt * ninst_);
        int tsc = 0;
        for (int i = 0; i < ninst_; ++i) {
            std::copy(inputs[i].R.begin(), inputs[i].R.end(), host.begin() + i * rt);
            tsc = std::max(tsc, inputs[i].tscale_log2);
        }
        if (const int st = upload(host.data(), tsc, err)) return st;
        CK(cudaStreamSynchronize(st_));
        return 0;
    }

    // R of every instance (ninst x tri(2n) entries of K doubles, the word type's layout) into
    // the resident level-0 buffers: one strided asynchronous copy on the plan's stream
    int upload(const double* R, int tscale_log2, std::string& err) override {
        if (const int st = upload_part(R, 0, ninst_, err)) return st;
        return upload_finish(tscale_log2, err);
    }
    // instances [lo, hi) of R (the whole batch's layout) -> device, asynchronously: callers
    // overlap building the next instances' R with the transfer of these
    int upload_part(const double* R, int lo, int hi, std::string& err) override {
        const size_t words = static_cast<size_t>(tri_sz(2 * n_)) * Arith<T>::K;
        CK(cudaSetDevice(device_));
        if (!up_started_.exchange(true)) CK(cudaEventRecord(ev_[4], st_));  // (debug timing) first copy
        CK(cudaMemcpyAsync(static_cast<double*>(rin_.p) + words * lo, R + words * lo, sizeof(double) * words * (hi - lo),
                           cudaMemcpyHostToDevice, st_));
        return 0;
    }
    int upload_finish(int tscale_log2, std::string& err) override {
        const size_t rt = static_cast<size_t>(tri_sz(2 * n_));
        tsc_ = tscale_log2;
        CK(cudaSetDevice(device_));
        // the contiguous upload (full link rate; a strided 2D copy of many instances runs row by
        // row) is scattered into the pool's per-instance buffers on the device
        {
            const uint64_t words = static_cast<uint64_t>(rt) * Arith<T>::K, total = words * ninst_;
            scatter_inputs_kernel<<<static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 1u << 20)), 256, 0,
                                    st_>>>(static_cast<const double*>(rin_.p), words, ninst_,
                                           static_cast<uint64_t>(g_.inst_entries) * Arith<T>::K,
                                           reinterpret_cast<double*>(pool()));
            CK(cudaGetLastError());
        }
        h2d_bytes_ = sizeof(T) * rt * ninst_;
        up_started_.store(false);
        return 0;
    }

    // Geometry and device buffers of `ninst` instances of n modes over `range` (no inputs).
    int init_geometry(int device, int n, int ninst, const WorkRange& range, std::string& err) {
        constexpr int Q0 = Cfg<T>::L + FAN;
        device_ = device;
        ninst_ = ninst;
        n_ = n;
        kbits_ = range.class_bits;
        clo_ = range.class_lo;
        chi_ = range.class_hi;
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
        for (auto& e : ev_) CK(cudaEventCreate(&e));
        if (const int st = ensure_ijtab(device, err)) return st;

        // Prefix depth c: a function of (n, instances) only -- not of this plan's class
        // range -- so every shard count evaluates the same jobs and the fixed fold tree
        // gives bit-identical results.  kWantJobs whole-problem jobs keep the dynamic
        // schedule's tail short even for the 1/8 shard of an 8-GPU run; job states are
        // <= kMaxJobModes modes.
        const uint64_t want_jobs = range.prefix_jobs ? range.prefix_jobs : (ninst_ > 1 ? kWantJobsBatch : kWantJobs);
        class_partials_ = range.class_partials;
        c_ = 0;
        if (n_ >= Q0) {
            int cw = 0;
            while ((static_cast<uint64_t>(ninst_) << cw) < want_jobs && cw < n_ - Q0) ++cw;
            c_ = std::max(cw, n_ - kMaxJobModes);
            c_ = std::min(c_, n_ - Q0);
            // Narrow slices (more than kShardBits class bits, e.g. checkpointed n = 50
            // pieces) deepen the prefix until the slice itself holds kWantJobs jobs; shards
            // of up to 2^kShardBits ranks keep the whole-problem depth (bit-identical folds).
            if (kbits_ > kShardBits) {
                int cs = kbits_;
                while (((chi_ - clo_) * static_cast<uint64_t>(ninst_) << (cs - kbits_)) < want_jobs && cs < n_ - Q0)
                    ++cs;
                c_ = std::max(c_, cs);
            }
        }
        use_levels_ = kbits_ <= c_;
        cj_ = use_levels_ ? c_ : kbits_;
        rjob_ = n_ - cj_;
        per_ = use_levels_ ? ((chi_ - clo_) << (c_ - kbits_)) : (chi_ - clo_);
        njobs_ = per_ * ninst_;

        g_ = PrefixGeom{};
        g_.n = n_;
        g_.c = use_levels_ ? c_ : 0;
        size_t o = tri_sz(2 * n_), to = 0;
        for (int e = 1; e <= g_.c; ++e) {
            // the level-e buffers under this plan's class range: the e-bit prefixes of
            // [lo, hi) ending in an include, p = prefix >> 1 (a contiguous range)
            const uint64_t lo = clo_ << (c_ - kbits_), hi = chi_ << (c_ - kbits_);
            const uint64_t plo = lo >> (c_ - e + 1), phi = (hi - 1) >> (c_ - e + 1);
            g_.plo[e] = plo;
            g_.off[e] = o;
            g_.toff[e] = to;
            o += (phi - plo + 1) * tri_sz(2 * (n_ - e));
            to += phi - plo + 1;
        }
        g_.inst_entries = o;
        g_.inst_ts = std::max<size_t>(to, 1);

        CK(pool_.alloc(sizeof(T) * g_.inst_entries * ninst_, device_));
        CK(tpool_.alloc(sizeof(T) * g_.inst_ts * ninst_, device_));
        CK(jobs_.alloc(sizeof(Job<T>) * njobs_, device_));
        CK(parts_.alloc(sizeof(double) * 5 * njobs_, device_));
        CK(errw_.alloc(sizeof(unsigned long long), device_));
        CK(res_.alloc(sizeof(double) * (static_cast<size_t>(ninst_) * 5 + 1), device_));
        // contiguous landing buffer of uploaded inputs (allocated here: upload_part may be
        // called from several host threads)
        CK(rin_.alloc(sizeof(T) * static_cast<size_t>(tri_sz(2 * n_)) * ninst_, device_));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&res_host_), sizeof(double) * (static_cast<size_t>(ninst_) * 5 + 1),
                         cudaHostAllocPortable));
        CK(ctr_.alloc(sizeof(unsigned long long), device_));
        if (!use_levels_) {
            work_stride_ = 2 * static_cast<size_t>(tri_sz(2 * n_));
            CK(work_.alloc(sizeof(T) * work_stride_ * njobs_, device_));
        }
        if (rjob_ >= Q0) {
            using SM = WarpSmem<T>;
            constexpr int WPB = Cfg<T>::WPB;
            smem_ = Cfg<T>::WS_MODE == 2 ? SM::kTabBytes + SM::kWarpBytes * 8 + sizeof(T) * SM::kProdEntries * 4
                                         : SM::kTabBytes + SM::kWarpBytes * (Cfg<T>::TSHARE ? WPB / 2 : WPB);
            for (auto* kfn : {subtree_kernel<T, false>, subtree_kernel<T, true>}) {
                CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
                CK(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            }
            int bps = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, subtree_kernel<T, false>, 32 * WPB, smem_));
            if (bps < 1) {
                err = "subtree kernel does not fit on an SM";
                return -1;
            }
            // The occupancy API reports 1 CTA/SM for kernels that allocate TMEM; two 4-warp
            // CTAs (256 TMEM columns each = the SM's 512) fit by registers and shared memory
            // and do run concurrently (measured: 264 -> 173 ms at n=32 DD).
            if (Cfg<T>::TMEM && Cfg<T>::WPB == 4 && 2 * (smem_ + 1024) <= 233472) bps = std::max(bps, 2);
            if (range.blocks_per_sm > 0) bps = range.blocks_per_sm;
            if (std::getenv("TOR_DEBUG_TIMING")) {
                cudaFuncAttributes fa;
                cudaFuncGetAttributes(&fa, subtree_kernel<T, false>);
                std::fprintf(stderr, "[tor] subtree_kernel: %d blocks/SM x %d warps, smem %zu B/block, %d regs, "
                                     "local %zu B, static smem %zu\n",
                             bps, WPB, smem_, fa.numRegs, fa.localSizeBytes, fa.sharedSizeBytes);
                for (size_t s2 : {size_t(0), size_t(50000), size_t(100000), size_t(110000), smem_}) {
                    int b2 = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, subtree_kernel<T, false>, 32 * WPB, s2);
                    size_t avail = 0;
                    cudaOccupancyAvailableDynamicSMemPerBlock(&avail, subtree_kernel<T, false>, 2, 32 * WPB);
                    std::fprintf(stderr, "[tor]   smem %zu -> %d blocks/SM (avail dyn smem @2 blocks: %zu)\n", s2, b2,
                                 avail);
                }
                cudaGetLastError();  // the availability query errors for TMEM kernels; not sticky
            }
            blocks_ = std::min<uint64_t>(static_cast<uint64_t>(bps) * sm_count_, (njobs_ + WPB - 1) / WPB);
            const int D = rjob_ - Q0;
            size_t stride = 0;
            for (int x = 1; x <= D; ++x) stride += tri_sz(2 * (rjob_ - x));
            scr_stride_ = std::max<size_t>(stride, 1);
            CK(scr_.alloc(sizeof(T) * scr_stride_ * blocks_ * WPB, device_));
        }
        return 0;
    }

    ~PlanImpl() override {
        if (graph_) cudaGraphExecDestroy(graph_);
        if (res_host_) cudaFreeHost(res_host_);
        for (auto& e : ev_)
            if (e) cudaEventDestroy(e);
        if (st_) cudaStreamDestroy(st_);
    }

    int execute(std::vector<EngineOut>& out, EngineStats* stats, std::string& err) override {
        if (const int st = launch(err)) return st;
        return collect(out, stats, err);
    }

    // Launch the whole device pipeline and the read-back on the plan's stream: the ~10-40
    // launches (memsets, prefix levels, jobs, subtree kernel, fold passes, gather, copy) are
    // captured once into a CUDA graph and replayed, so a repeated small evaluation pays one
    // launch (the graph is re-captured when the input scaling selects the other kernel).
    int launch(std::string& err) override {
        CK(cudaSetDevice(device_));
        const auto tx0 = std::chrono::steady_clock::now();
        if (!graph_ || graph_tsc_ != tsc_) {
            if (graph_) {
                cudaGraphExecDestroy(graph_);
                graph_ = nullptr;
            }
            cudaGraph_t g = nullptr;
            CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
            const int st = enqueue(err);
            const cudaError_t ce = cudaStreamEndCapture(st_, &g);
            if (st != 0) {
                if (g) cudaGraphDestroy(g);
                return st;
            }
            CK(ce);
            const cudaError_t ie = cudaGraphInstantiate(&graph_, g, 0);
            cudaGraphDestroy(g);
            CK(ie);
            graph_tsc_ = tsc_;
        }
        CK(cudaGraphLaunch(graph_, st_));
        tx0_ = tx0;
        return 0;
    }

    // the pipeline's work on st_ (captured by launch)
    int enqueue(std::string& err) {
        constexpr int Q0 = Cfg<T>::L + FAN;
        uint64_t launches = 0;
        unsigned long long* errw = static_cast<unsigned long long*>(errw_.p);
        unsigned long long* ctr = static_cast<unsigned long long*>(ctr_.p);
        double* parts = static_cast<double*>(parts_.p);
        Job<T>* jobs = static_cast<Job<T>*>(jobs_.p);
        CK(cudaMemsetAsync(errw, 0xff, sizeof(unsigned long long), st_));
        CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st_));
        CK(cudaEventRecordWithFlags(ev_[0], st_, cudaEventRecordExternal));
        if (use_levels_) {
            const int wpb = 4;
            const size_t sm = sizeof(T) * 4 * n_ * wpb;
            const uint64_t lo = clo_ << (c_ - kbits_), hi = chi_ << (c_ - kbits_);
            for (int e = 1; e <= g_.c; ++e) {
                // only the level-e buffers under this plan's class range (PrefixGeom::plo)
                const uint64_t plo = g_.plo[e], phi = (hi - 1) >> (c_ - e + 1);
                const uint64_t cnt = phi - plo + 1;
                const uint64_t items = cnt * ninst_;
                // few nodes: several warps per elimination (>= 128 trailing entries each)
                const int tot = tri_sz(2 * (n_ - e));
                int parts = 1;
                while (parts < 32 && items * parts * 2 <= static_cast<uint64_t>(sm_count_) * 8 &&
                       tot / (parts * 2) >= 128)
                    parts *= 2;
                const uint64_t blocks = std::min<uint64_t>((items * parts + wpb - 1) / wpb, 65535ull * 4);
                prefix_level_kernel<T><<<static_cast<unsigned>(blocks), 32 * wpb, sm, st_>>>(
                    g_, pool(), tpool(), e, ninst_, plo, cnt, parts, errw);
                ++launches;
            }
            const uint64_t blocks = std::min<uint64_t>((njobs_ + 255) / 256, 1ull << 20);
            make_jobs_kernel<T><<<static_cast<unsigned>(blocks), 256, 0, st_>>>(g_, pool(), tpool(), ninst_, lo, hi,
                                                                                jobs);
            ++launches;
        } else {
            const int wpb = 4;
            const size_t sm = sizeof(T) * (4 * n_ * wpb + wpb);
            const uint64_t blocks = std::min<uint64_t>((njobs_ + wpb - 1) / wpb, 65535ull * 4);
            direct_prefix_kernel<T><<<static_cast<unsigned>(blocks), 32 * wpb, sm, st_>>>(
                n_, kbits_, pool(), ninst_, g_.inst_entries, clo_, chi_, static_cast<T*>(work_.p), work_stride_, jobs,
                errw);
            ++launches;
        }
        CK(cudaGetLastError());
        CK(cudaEventRecordWithFlags(ev_[1], st_, cudaEventRecordExternal));
        if (rjob_ >= Q0) {
            constexpr int WPB = Cfg<T>::WPB;
            auto* kfn = tsc_ ? subtree_kernel<T, true> : subtree_kernel<T, false>;
            kfn<<<static_cast<unsigned>(blocks_), 32 * WPB, smem_, st_>>>(jobs, njobs_, n_, rjob_,
                                                                          static_cast<T*>(scr_.p), scr_stride_, parts,
                                                                          errw, ctr, tsc_);
        } else {
            const uint64_t blocks = (njobs_ + 127) / 128;
            small_job_kernel<T, Q0 - 1><<<static_cast<unsigned>(blocks), 128, 0, st_>>>(jobs, njobs_, n_, rjob_,
                                                                                        parts, errw, tsc_);
        }
        ++launches;
        CK(cudaGetLastError());
        CK(cudaEventRecordWithFlags(ev_[2], st_, cudaEventRecordExternal));
        // jobs per output partial: the whole range, or one class (a power of two)
        const uint64_t chunk = class_partials_ ? per_ / (chi_ - clo_) : per_;
        for (uint64_t S = 1; S < chunk; S *= kFoldB) {
            const uint64_t cnt = (per_ + S - 1) / S;
            const int G = class_partials_ ? static_cast<int>(std::min<uint64_t>(kFoldB, chunk / S)) : kFoldB;
            for (int i0 = 0; i0 < ninst_; i0 += 65535) {
                const int ni = std::min(ninst_ - i0, 65535);
                fold_pass_kernel<T><<<dim3(static_cast<unsigned>((cnt + kFoldB - 1) / kFoldB), ni), kFoldB / 2, 0,
                                      st_>>>(parts, per_, S, i0, G);
                ++launches;
            }
        }
        CK(cudaGetLastError());
        CK(cudaEventRecordWithFlags(ev_[3], st_, cudaEventRecordExternal));
        double* resd = static_cast<double*>(res_.p);
        gather_results_kernel<<<static_cast<unsigned>((ninst_ * 5 + 255) / 256), 256, 0, st_>>>(parts, per_, ninst_,
                                                                                              errw, resd);
        ++launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(res_host_, resd, sizeof(double) * (static_cast<size_t>(ninst_) * 5 + 1),
                           cudaMemcpyDeviceToHost, st_));
        CK(cudaEventRecordWithFlags(ev_[5], st_, cudaEventRecordExternal));
        launches_ = launches;
        return 0;
    }

    // wait for the launched pipeline and decode its results
    int collect(std::vector<EngineOut>& out, EngineStats* stats, std::string& err) override {
        CK(cudaSetDevice(device_));
        const uint64_t launches = launches_;
        const auto tx0 = tx0_;
        double* parts = static_cast<double*>(parts_.p);
        const uint64_t chunk = class_partials_ ? per_ / (chi_ - clo_) : per_;
        const double* res = res_host_;
        std::vector<double> cls;
        if (class_partials_) {
            const uint64_t ncls = chi_ - clo_;
            cls.resize(static_cast<size_t>(ninst_) * ncls * 5);
            for (int i = 0; i < ninst_; ++i)
                CK(cudaMemcpy2DAsync(cls.data() + i * ncls * 5, 5 * sizeof(double), parts + i * per_ * 5,
                                     chunk * 5 * sizeof(double), 5 * sizeof(double), ncls, cudaMemcpyDeviceToHost,
                                     st_));
        }
        const auto tq = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(st_));
        if (std::getenv("TOR_DEBUG_TIMING")) {
            float up = 0, dn = 0, dv = 0;
            cudaEventElapsedTime(&up, ev_[4], ev_[0]);
            cudaEventElapsedTime(&dv, ev_[0], ev_[3]);
            cudaEventElapsedTime(&dn, ev_[3], ev_[5]);
            std::fprintf(stderr, "[tor] events: upload..start %.3f ms, pipeline %.3f ms, gather+readback %.3f ms\n", up,
                         dv, dn);
            std::fprintf(stderr, "[tor] execute: enqueue %.3f ms, sync wait %.3f ms\n",
                         std::chrono::duration<double, std::milli>(tq - tx0).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq).count());
        }
        unsigned long long herr;
        std::memcpy(&herr, res + static_cast<size_t>(ninst_) * 5, sizeof(herr));
        out.assign(ninst_, EngineOut{});
        const uint64_t terms = (chi_ - clo_) << (n_ - kbits_);
        for (int i = 0; i < ninst_; ++i) {
            for (int x = 0; x < 4; ++x) out[i].words[x] = res[i * 5 + x];
            out[i].sum_abs = res[i * 5 + 4];
            out[i].terms = terms;
            if (class_partials_) {
                // the classes, and the range's total folded from them on the host
                const size_t ncls = chi_ - clo_;
                out[i].class_parts.assign(cls.begin() + i * ncls * 5, cls.begin() + (i + 1) * ncls * 5);
                double w5[5];
                fold_words(std::is_same<T, qd>::value ? MODE_QD : MODE_DD, out[i].class_parts.data(),
                           static_cast<int>(ncls), w5);
                for (int x = 0; x < 4; ++x) out[i].words[x] = w5[x];
                out[i].sum_abs = w5[4];
            }
            if (herr != ~0ull) {
                out[i].breakdown = true;
                out[i].bad_mask = herr >> 8;
                out[i].bad_row = static_cast<int>(herr & 0xff);
            }
        }
        if (stats) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, ev_[1], ev_[2]);
            cudaEventElapsedTime(&b, ev_[0], ev_[3]);
            stats->kernel_ms = a;
            stats->total_ms = b;
            stats->launches = launches;
            stats->prefix_depth = cj_;
            stats->jobs = njobs_;
            stats->h2d_bytes = h2d_bytes_;
            stats->d2h_bytes = (static_cast<size_t>(ninst_) * 5 + cls.size()) * sizeof(double) + sizeof(herr);
        }
        return 0;
    }

  private:
    T* pool() { return static_cast<T*>(pool_.p); }
    T* tpool() { return static_cast<T*>(tpool_.p); }
    int device_ = 0, ninst_ = 0, n_ = 0, kbits_ = 0, sm_count_ = 0, c_ = 0, cj_ = 0, rjob_ = 0, tsc_ = 0;
    uint64_t clo_ = 0, chi_ = 1, per_ = 0, njobs_ = 0, blocks_ = 0;
    bool use_levels_ = true, class_partials_ = false;
    PrefixGeom g_{};
    size_t smem_ = 0, scr_stride_ = 1, work_stride_ = 0, h2d_bytes_ = 0;
    cudaStream_t st_ = nullptr;
    cudaEvent_t ev_[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    std::atomic<bool> up_started_{false};
    DevBuf pool_, tpool_, jobs_, parts_, errw_, ctr_, scr_, work_, res_, rin_;
    double* res_host_ = nullptr;  // pinned: ninst x 5 result words + the breakdown word
    uint64_t launches_ = 0;       // kernels in the launched graph
    cudaGraphExec_t graph_ = nullptr;
    int graph_tsc_ = -1;
    std::chrono::steady_clock::time_point tx0_;
};

template <class T>
int make_plan(int device, const std::vector<PreparedInput>& inputs, const WorkRange& range, Plan** out,
              std::string& err) {
    auto* p = new PlanImpl<T>();
    const int st = p->init(device, inputs, range, err);
    if (st != 0) {
        delete p;
        return st;
    }
    *out = p;
    return 0;
}

}  // namespace

void release_staged_cache();
void release_device_cache() {
    release_staged_cache();
    DevPool& pl = DevPool::get();
    std::lock_guard<std::mutex> lk(pl.mu);
    for (int d = 0; d < 64; ++d) {
        if (pl.free_blocks[d].empty()) continue;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(d);
        for (auto& kv : pl.free_blocks[d]) cudaFree(kv.second);
        pl.free_blocks[d].clear();
        pl.pooled[d] = 0;
        cudaSetDevice(cur);
    }
}

int engine_tree_min_n(int mode) {
    return mode == MODE_QD ? Cfg<qd>::L + FAN : (mode == MODE_DD ? Cfg<dd>::L + FAN : Cfg<double>::L + FAN);
}

namespace {
template <class T>
int make_geometry(int device, int n, int ninst, const WorkRange& range, Plan** out, std::string& err) {
    auto* p = new PlanImpl<T>();
    const int st = p->init_geometry(device, n, ninst, range, err);
    if (st != 0) {
        delete p;
        return st;
    }
    *out = p;
    return 0;
}

bool same_range(const WorkRange& a, const WorkRange& b) {
    return a.class_bits == b.class_bits && a.class_lo == b.class_lo && a.class_hi == b.class_hi &&
           a.class_partials == b.class_partials && a.prefix_jobs == b.prefix_jobs && a.blocks_per_sm == b.blocks_per_sm;
}

// Process-wide cache of idle staged plans (device buffers, stream, events, pinned staging),
// least recently used last; an acquired plan is owned by its caller until released.
struct StagedCache {
    static constexpr size_t kMax = 6;
    std::mutex mu;
    std::vector<StagedPlan*> idle;
    static StagedCache& get() {
        static StagedCache c;
        return c;
    }
};
}  // namespace

StagedPlan::~StagedPlan() {
    delete plan;
    if (staging) cudaFreeHost(staging);
}

int staged_acquire(int device, int mode, int n, int count, const WorkRange& range, StagedPlan** out,
                   std::string& err) {
    *out = nullptr;
    {
        StagedCache& c = StagedCache::get();
        std::lock_guard<std::mutex> lk(c.mu);
        for (size_t i = 0; i < c.idle.size(); ++i) {
            StagedPlan* sp = c.idle[i];
            if (sp->device == device && sp->mode == mode && sp->n == n && sp->count == count &&
                same_range(sp->range, range)) {
                c.idle.erase(c.idle.begin() + static_cast<long>(i));
                *out = sp;
                return 0;
            }
        }
    }
    auto* sp = new StagedPlan();
    sp->device = device;
    sp->mode = mode;
    sp->n = n;
    sp->count = count;
    sp->range = range;
    const int st = mode == MODE_FP64 ? make_geometry<double>(device, n, count, range, &sp->plan, err)
                   : mode == MODE_DD ? make_geometry<dd>(device, n, count, range, &sp->plan, err)
                                     : make_geometry<qd>(device, n, count, range, &sp->plan, err);
    if (st != 0) {
        delete sp;
        return st;
    }
    sp->stride = static_cast<size_t>(2 * n) * (2 * n + 1) / 2 * mode_words(mode);
    const cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&sp->staging), sizeof(double) * sp->stride * count,
                                        cudaHostAllocPortable);
    if (e != cudaSuccess) {
        err = std::string("cudaHostAlloc: ") + cudaGetErrorString(e);
        delete sp;
        return static_cast<int>(e);
    }
    *out = sp;
    return 0;
}

int staged_execute(StagedPlan* sp, int tscale_log2, std::vector<EngineOut>& out, EngineStats* stats,
                   std::string& err) {
    const auto t0 = std::chrono::steady_clock::now();
    if (const int st = sp->plan->upload(sp->staging, tscale_log2, err)) return st;
    const auto t1 = std::chrono::steady_clock::now();
    const int st = sp->plan->execute(out, stats, err);
    if (std::getenv("TOR_DEBUG_TIMING")) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[tor] staged: upload enqueue %.3f ms, execute %.3f ms (device %.3f ms)\n", ms(t0, t1),
                     ms(t1, std::chrono::steady_clock::now()), stats ? stats->total_ms : -1.0);
    }
    return st;
}

int staged_upload_part(StagedPlan* sp, int lo, int hi, std::string& err) {
    return sp->plan->upload_part(sp->staging, lo, hi, err);
}

int staged_execute_uploaded(StagedPlan* sp, int tscale_log2, std::vector<EngineOut>& out, EngineStats* stats,
                            std::string& err) {
    if (const int st = staged_launch(sp, tscale_log2, err)) return st;
    return staged_collect(sp, out, stats, err);
}

int staged_launch(StagedPlan* sp, int tscale_log2, std::string& err) {
    if (const int st = sp->plan->upload_finish(tscale_log2, err)) return st;
    return sp->plan->launch(err);
}

int staged_collect(StagedPlan* sp, std::vector<EngineOut>& out, EngineStats* stats, std::string& err) {
    return sp->plan->collect(out, stats, err);
}

void staged_release(StagedPlan* sp) {
    if (!sp) return;
    StagedCache& c = StagedCache::get();
    std::vector<StagedPlan*> drop;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        c.idle.insert(c.idle.begin(), sp);
        while (c.idle.size() > StagedCache::kMax) {
            drop.push_back(c.idle.back());
            c.idle.pop_back();
        }
    }
    for (auto* d : drop) delete d;
}

void release_staged_cache() {
    StagedCache& c = StagedCache::get();
    std::vector<StagedPlan*> drop;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        drop.swap(c.idle);
    }
    for (auto* d : drop) delete d;
}

int plan_create(int device, int mode, const std::vector<PreparedInput>& inputs, const WorkRange& range, Plan** out,
                std::string& err) {
    *out = nullptr;
    if (inputs.empty()) {
        err = "no inputs";
        return -1;
    }
    switch (mode) {
        case MODE_FP64:
            return make_plan<double>(device, inputs, range, out, err);
        case MODE_DD:
            return make_plan<dd>(device, inputs, range, out, err);
        case MODE_QD:
            return make_plan<qd>(device, inputs, range, out, err);
        default:
            err = "bad mode";
            return -1;
    }
}

int engine_run(int device, int mode, const std::vector<PreparedInput>& inputs, const WorkRange& range,
               std::vector<EngineOut>& out, EngineStats* stats, std::string& err) {
    if (inputs.empty()) {
        out.clear();
        return 0;
    }
    Plan* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const int st = plan_create(device, mode, inputs, range, &p, err);
    if (st != 0) return st;
    const auto t1 = std::chrono::steady_clock::now();
    const int rs = p->execute(out, stats, err);
    const auto t2 = std::chrono::steady_clock::now();
    delete p;
    if (std::getenv("TOR_DEBUG_TIMING")) {
        const auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[tor] engine_run: plan_create %.3f ms, execute %.3f ms, destroy %.3f ms\n", ms(t0, t1),
                     ms(t1, t2), ms(t2, t3));
    }
    return rs;
}

namespace {
// fold of the aligned blocks covering classes [a, a + w) along the fixed tree
bool fold_range(int mode, const double* parts, const uint64_t* lo, const uint64_t* width, int count, uint64_t a,
                uint64_t w, int& next, double* out5) {
    if (next >= count || lo[next] < a) return false;
    if (lo[next] == a && width[next] == w) {
        for (int x = 0; x < 5; ++x) out5[x] = parts[5 * next + x];
        ++next;
        return true;
    }
    if (w == 1 || lo[next] != a || width[next] > w) return false;
    double r[5];
    if (!fold_range(mode, parts, lo, width, count, a, w / 2, next, out5)) return false;
    if (!fold_range(mode, parts, lo, width, count, a + w / 2, w / 2, next, r)) return false;
    if (mode == MODE_QD) merge_words<qd>(out5, r);
    else merge_words<dd>(out5, r);
    return true;
}
}  // namespace

bool fold_blocks(int mode, const double* parts, const uint64_t* lo, const uint64_t* width, int count,
                 int class_bits, double* out5) {
    if (count < 1 || class_bits < 0 || class_bits > 62) return false;
    for (int i = 0; i < count; ++i)
        if (width[i] == 0 || (width[i] & (width[i] - 1)) || lo[i] % width[i]) return false;
    int next = 0;
    return fold_range(mode, parts, lo, width, count, 0, 1ull << class_bits, next, out5) && next == count;
}

void fold_words(int mode, const double* parts, int count, double* out5) {
    // same pairwise tree as fold_pass_kernel over `count` shard partials (5 doubles each)
    std::vector<double> p(parts, parts + 5 * static_cast<size_t>(count));
    for (int s = 1; s < count; s <<= 1)
        for (int i = 0; i + s < count; i += 2 * s) {
            if (mode == MODE_QD) merge_words<qd>(&p[5 * i], &p[5 * (i + s)]);
            else merge_words<dd>(&p[5 * i], &p[5 * (i + s)]);
        }
    for (int i = 0; i < 5; ++i) out5[i] = count ? p[i] : 0.0;
}

}  // namespace tor
