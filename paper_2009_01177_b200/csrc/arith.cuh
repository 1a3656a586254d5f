// Multi-word floating-point arithmetic on FP64 FMA for the Torontonian engine.
//
// Replaces the reference's fixed-point Wide<W> limbs (fixed_point.hpp:27-160,
// fixed_point.cpp:52-162): the 128-bit mode becomes double-double (DD, 2 x f64,
// ~106-bit significand) and the 256-bit mode quad-double (QD, 4 x f64, ~212-bit),
// both unevaluated sums built from error-free transformations (TwoSum, TwoProd
// via DFMA).  Floating words keep RELATIVE precision, so the reference's
// global-scaling failure modes (fixed-point BreakdownError on tiny pivots,
// test_torontonian.cpp:218-244) do not occur; only a truly non-positive pivot
// breaks down.
//
// Build contract: compiled with --fmad=false (device) / -ffp-contract=off (host),
// so every `a*b + c` below is two roundings unless written as fma() explicitly.
// The ops and their FP64 instruction counts are pinned in profiles/sass_counts.json.
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define TOR_UNROLL _Pragma("unroll")
#define TOR_HD __host__ __device__ __forceinline__
// large QD routines: inline (measured faster than out-of-line calls even though the QD
// kernel's SASS is ~60K instructions)
#define TOR_HD_NI TOR_HD
// QD rank-1/rank-2 entry updates as out-of-line calls (one copy each): measured
// 407 -> 352 ms at n=28 QD (instruction-cache bound kernel); -DTOR_QD_RANK_INLINE inlines
// them (used only by the arithmetic probes of tools/probes/prims.cu, which count the bodies)
#ifndef TOR_QD_RANK_INLINE
#define TOR_HD_RNI __host__ __device__ __noinline__
#else
#define TOR_HD_RNI TOR_HD
#endif
#else
#define TOR_UNROLL
#define TOR_HD inline
#define TOR_HD_NI inline
#define TOR_HD_RNI inline
#endif

namespace tor {

// ---------------------------------------------------------------- helpers --
TOR_HD double fma_(double a, double b, double c) { return fma(a, b, c); }

// Error-free transformations.
TOR_HD void two_sum(double a, double b, double& s, double& e) {
    s = a + b;
    const double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}
// Requires exponent(a) >= exponent(b) (or a == 0).
TOR_HD void fast_two_sum(double a, double b, double& s, double& e) {
    s = a + b;
    e = b - (s - a);
}
TOR_HD void two_prod(double a, double b, double& p, double& e) {
    p = a * b;
    e = fma_(a, b, -p);
}

// Non-positive (or -0/+0) test on the high word: integer pipe, no FP64 issue slot.
TOR_HD bool nonpositive(double x) {
#if defined(__CUDA_ARCH__)
    return __double2hiint(x) <= 0;
#else
    return !(x > 0.0);
#endif
}

// fp64 reciprocal square root seed: MUFU.RSQ64H (~2^-23 relative).  The host build
// (arithmetic unit tests) emulates the seed's accuracy by truncating 1/sqrt(x) to its
// leading 20 significand bits, so the Newton steps below run on the same path.
TOR_HD double rsqrt_seed(double x) {
#if defined(__CUDA_ARCH__)
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
#else
    int e;
    const double f = std::frexp(1.0 / std::sqrt(x), &e);
    return std::ldexp(std::floor(std::ldexp(f, 20)), e - 20);
#endif
}
// Two fp64 Newton steps from the seed y ~ 1/sqrt(x) -> ~1 ulp.  The seed may come from
// an approximation of x (e.g. an unnormalised leading word): the steps converge to
// 1/sqrt(x) for any seed within a few 2^-20 of it.
TOR_HD double rsqrt_newton(double x, double y) {
    // one third-order step y (1 + r/2 + 3 r^2 / 8), r = 1 - x y^2: from a 2^-20 seed the
    // truncation error is ~(5/16) r^3 < 2^-58, i.e. the result is fp64-rounding-limited
    // (~1 ulp) after 4 dependent operations instead of 6 for two Newton steps
    const double r = fma_(-x, y * y, 1.0);
    const double p = fma_(0.375, r, 0.5);
    return fma_(y * r, p, y);
}
// Full-precision fp64 reciprocal square root for x > 0.
TOR_HD double rsqrt_d(double x) { return rsqrt_newton(x, rsqrt_seed(x)); }

// ===================================================================== DD ==
struct dd {
    double hi, lo;
};

TOR_HD dd dd_make(double x) { return dd{x, 0.0}; }

// Renormalise an arbitrary (h, l) pair exactly (TwoSum: no ordering assumption).
TOR_HD dd dd_norm(dd a) {
    dd r;
    two_sum(a.hi, a.lo, r.hi, r.lo);
    return r;
}

TOR_HD dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }

// Product of two DD values, normalised.  a may be unnormalised (h, l) with small l.
TOR_HD dd dd_mul(dd a, dd b) {
    double p, e;
    two_prod(a.hi, b.hi, p, e);
    e = fma_(a.hi, b.lo, e);
    e = fma_(a.lo, b.hi, e);
    dd r;
    fast_two_sum(p, e, r.hi, r.lo);
    return r;
}

// Accurate sum (both TwoSums, IEEE-style DD add): relative error ~2^-104 of the result.
TOR_HD dd dd_add(dd a, dd b) {
    double s, e, t, f;
    two_sum(a.hi, b.hi, s, e);
    two_sum(a.lo, b.lo, t, f);
    e += t;
    fast_two_sum(s, e, s, e);
    e += f;
    dd r;
    fast_two_sum(s, e, r.hi, r.lo);
    return r;
}
TOR_HD dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

// Lazy symmetric rank-2 update entry  s - a*b - c*d.  s may be unnormalised; the
// result is the exact hi part of the TwoSum chain plus an un-renormalised lo.
// Backward-stable at the DD level: |err| <= O(2^-105) (|s| + |ab| + |cd|).
TOR_HD dd dd_rank2(dd s, dd a, dd b, dd c, dd d) {
    double p1, e1, p2, e2, s1, f1, s2, f2;
    two_prod(a.hi, b.hi, p1, e1);
    two_prod(c.hi, d.hi, p2, e2);
    two_sum(s.hi, -p1, s1, f1);
    two_sum(s1, -p2, s2, f2);
    double lo = s.lo + f1;
    lo = lo + f2;
    lo = lo - e1;
    lo = lo - e2;
    lo = fma_(-a.hi, b.lo, lo);
    lo = fma_(-a.lo, b.hi, lo);
    lo = fma_(-c.hi, d.lo, lo);
    lo = fma_(-c.lo, d.hi, lo);
    return dd{s2, lo};
}
// s - a*b (lazy, as above).
TOR_HD dd dd_rank1(dd s, dd a, dd b) {
    double p1, e1, s1, f1;
    two_prod(a.hi, b.hi, p1, e1);
    two_sum(s.hi, -p1, s1, f1);
    double lo = s.lo + f1;
    lo = lo - e1;
    lo = fma_(-a.hi, b.lo, lo);
    lo = fma_(-a.lo, b.hi, lo);
    return dd{s1, lo};
}

// ---- fixed-exponent (biased grid) DD for Schur-complement states -----------------
// Every entry of every Schur complement of the (scaled) R satisfies |S_ij| <= max_k R_kk
// (SPD: Schur complements only shrink the diagonal, |S_ij| <= sqrt(S_ii S_jj)), and so do
// the partial complements S - u u^T and the Cholesky products |u_i u_j|, |w_i w_j|.  With
// max_k R_kk < 3.75 a state entry is stored BIASED: its leading word is b = s_hi + C with
// C = 12, so b lies in [8.25, 15.75] where the double spacing is 2^-kGridG -- the leading
// word sits on the grid 2^-49 by construction.  A rank-2 entry update is then
//     z1 = fma(-u_i, u_j, b)      (= grid(s - u_i u_j) + C: the FMA rounds onto the grid)
//     r1 = fma(u_i, u_j, z1 - b)  (the product's grid remainder; z1 - b exact)
//     z2 = fma(-w_i, w_j, z1),  r2 = fma(w_i, w_j, z2 - z1)
// and the low word collects s_lo - r1 - r2 and the four cross products: 12 FP64
// instructions per entry (8 DFMA, 4 DADD) instead of 16 for an unbiased grid (DMUL +
// two DADDs per grid rounding) or 24 with TwoSums.  Same backward error shape (absolute,
// ~2^-103 of the O(1) state scale).  Values leave the biased form (unb(): one exact
// DADD) only where they become pivots or pivot-row vectors.
constexpr int kGridG = 49;
constexpr double kGridC = 12.0;  // 1.5 * 2^(52 - kGridG): s + C lies in [8, 16) for |s| < 4

TOR_HD double grid_round(double p) { return (p + kGridC) - kGridC; }

// (x + y) as a biased grid state entry (host-side R construction)
TOR_HD dd dd_to_grid(double x, double y) {
    double sh, se;
    two_sum(x, y, sh, se);
    const double B = sh + kGridC;  // rounds sh onto the grid (exact in [8, 16))
    return dd{B, (sh - (B - kGridC)) + se};
}
TOR_HD dd dd_unbias(const dd& s) { return dd{s.hi - kGridC, s.lo}; }

TOR_HD dd dd_rank2_grid(dd s, dd a, dd b, dd c, dd d) {
    const double z1 = fma_(-a.hi, b.hi, s.hi);
    const double r1 = fma_(a.hi, b.hi, z1 - s.hi);
    const double z2 = fma_(-c.hi, d.hi, z1);
    const double r2 = fma_(c.hi, d.hi, z2 - z1);
    double lo = s.lo - r1;
    lo = lo - r2;
    lo = fma_(-a.hi, b.lo, lo);
    lo = fma_(-a.lo, b.hi, lo);
    lo = fma_(-c.hi, d.lo, lo);
    lo = fma_(-c.lo, d.hi, lo);
    return dd{z2, lo};
}
// s - a*b for a biased state entry s (the partial complement of a pivot-row vector);
// the result is UNBIASED (it feeds a product)
TOR_HD dd dd_rank1_grid(dd s, dd a, dd b) {
    const double z1 = fma_(-a.hi, b.hi, s.hi);
    const double r1 = fma_(a.hi, b.hi, z1 - s.hi);
    double lo = s.lo - r1;
    lo = fma_(-a.hi, b.lo, lo);
    lo = fma_(-a.lo, b.hi, lo);
    return dd{z1 - kGridC, lo};
}

// 1/sqrt(x) for normalised x > 0 from the fp64 seed y0 (of x.hi or an approximation
// of it): fp64 Newton to ~1 ulp, then one DD Newton step on the exact residual
// r = 1 - x*y^2 (y^2 exact by TwoProd).  Result is (y, y*r/2), |lo| <= ulp.
TOR_HD dd dd_rsqrt_seeded(dd x, double y0) {
    const double y = rsqrt_newton(x.hi, y0);
    double p, pe;
    two_prod(y, y, p, pe);
    double r = fma_(-x.hi, p, 1.0);
    r = fma_(-x.hi, pe, r);
    r = fma_(-x.lo, p, r);
    const double c = (0.5 * y) * r;
    return dd{y, c};
}
TOR_HD dd dd_rsqrt(dd x) { return dd_rsqrt_seeded(x, rsqrt_seed(x.hi)); }

// det [[a, b], [b, c]] = a c - b^2 for DD a, b, c (possibly un-normalised): TwoProds of
// the leading words, ONE TwoSum for the (possibly cancelling) difference, the cross
// products into the low word, then a fast renormalisation.  h (the rounded leading difference, available a few
// operations in) is a good enough seed argument for the reciprocal square root.
TOR_HD dd dd_det2(const dd& a, const dd& b, const dd& c, double& h) {
    const double p = a.hi * c.hi;
    const double pe = fma_(a.hi, c.hi, -p);
    const double q = b.hi * b.hi;
    const double qe = fma_(b.hi, b.hi, -q);
    double he;
    two_sum(p, -q, h, he);
    double t = fma_(a.hi, c.lo, a.lo * c.hi);
    t = fma_(-2.0 * b.hi, b.lo, t);
    const double lo = (he + (pe - qe)) + t;
    dd r;
    fast_two_sum(h, lo, r.hi, r.lo);
    return r;
}

// ===================================================================== QD ==
// Four non-overlapping doubles x0 > x1 > x2 > x3 (Hida-Li-Bailey style algorithms,
// restated from their published error-free-transformation formulation).
struct qd {
    double x[4];
};

TOR_HD qd qd_make(double a) { return qd{{a, 0.0, 0.0, 0.0}}; }
TOR_HD qd qd_neg(qd a) { return qd{{-a.x[0], -a.x[1], -a.x[2], -a.x[3]}}; }

// Branch-free renormalisation: two cascaded passes of TwoSum (exact for any
// ordering), result non-overlapping up to a few ulps -- adequate for the engine's
// 2^-180 budget and SIMT friendly (no data-dependent branches).
TOR_HD qd qd_renorm5_bf(double c0, double c1, double c2, double c3, double c4) {
    // pass 1: bottom-up accumulation
    double e3, e2, e1, e0;
    two_sum(c3, c4, c3, e3);
    two_sum(c2, c3, c2, e2);
    two_sum(c1, c2, c1, e1);
    two_sum(c0, c1, c0, e0);
    // now c0 holds the leading value; e0..e3 the errors in decreasing magnitude
    double t0, t1, t2;
    two_sum(e0, e1, t0, t1);
    two_sum(t1, e2, t1, t2);
    t2 += e3;
    double r0, r1, r2, r3;
    two_sum(c0, t0, r0, t0);
    two_sum(t0, t1, r1, t1);
    two_sum(t1, t2, r2, r3);
    return qd{{r0, r1, r2, r3}};
}

// One-pass renormalisation of order-collected words h0..h3 (h_k ~ 2^-53k of the operands'
// scale): a chain of three TwoSums (exact for any ordering -- a lazy state-entry operand may
// have cancelled its leading word).  The words come out at most their nominal order 2^-53k
// of that scale, which is all the order-collected operations that consume them assume; the
// full two-pass renormalisation is kept where a value must be normalised relative to ITSELF
// (pivots, determinants, the rsqrt residual).
TOR_HD qd qd_renorm_lead(double h0, double h1, double h2, double h3) {
    double s0, e1, s1, e2, s2, s3;
    two_sum(h0, h1, s0, e1);
    two_sum(e1, h2, s1, e2);
    two_sum(e2, h3, s2, s3);
    return qd{{s0, s1, s2, s3}};
}
TOR_HD void three_sum(double& a, double& b, double& c) {
    double t1, t2, t3;
    two_sum(a, b, t1, t2);
    two_sum(c, t1, a, t3);
    two_sum(t2, t3, b, c);
}
TOR_HD void three_sum2(double& a, double& b, double c) {
    double t1, t2, t3;
    two_sum(a, b, t1, t2);
    two_sum(c, t1, a, t3);
    b = t2 + t3;
}

// Accurate-enough QD addition ("sloppy" add: pairwise TwoSums then renormalise).
TOR_HD_NI qd qd_add(qd a, qd b) {
    double s0, s1, s2, s3, t0, t1, t2, t3;
    two_sum(a.x[0], b.x[0], s0, t0);
    two_sum(a.x[1], b.x[1], s1, t1);
    two_sum(a.x[2], b.x[2], s2, t2);
    two_sum(a.x[3], b.x[3], s3, t3);
    two_sum(s1, t0, s1, t0);
    three_sum(s2, t0, t1);
    three_sum2(s3, t0, t2);
    t0 = t0 + t1 + t3;
    return qd_renorm5_bf(s0, s1, s2, s3, t0);
}
TOR_HD qd qd_sub(const qd& a, const qd& b) { return qd_add(a, qd_neg(b)); }

// QD product (sloppy: terms of order >= 4 in the component index dropped).
TOR_HD_NI qd qd_mul(qd a, qd b) {
    double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5;
    double t0, t1, s0, s1, s2;
    two_prod(a.x[0], b.x[0], p0, q0);
    two_prod(a.x[0], b.x[1], p1, q1);
    two_prod(a.x[1], b.x[0], p2, q2);
    two_prod(a.x[0], b.x[2], p3, q3);
    two_prod(a.x[1], b.x[1], p4, q4);
    two_prod(a.x[2], b.x[0], p5, q5);
    // order 1
    three_sum(p1, p2, q0);
    // order 2: p2, q1, q2, p3, p4, p5
    three_sum(p2, q1, q2);
    three_sum(p3, p4, p5);
    two_sum(p2, p3, s0, t0);
    two_sum(q1, p4, s1, t1);
    s2 = q2 + p5;
    two_sum(s1, t0, s1, t0);
    s2 += (t0 + t1);
    // order 3
    s1 += a.x[0] * b.x[3] + a.x[1] * b.x[2] + a.x[2] * b.x[1] + a.x[3] * b.x[0] + q0 + q3 + q4 +
          q5;
    return qd_renorm5_bf(p0, p1, s0, s1, s2);
}

// QD x double.
TOR_HD qd qd_mul_d(const qd& a, double b) {
    double p0, p1, p2, p3, q0, q1, q2, s0, s1, s2, s3, s4;
    two_prod(a.x[0], b, p0, q0);
    two_prod(a.x[1], b, p1, q1);
    two_prod(a.x[2], b, p2, q2);
    p3 = a.x[3] * b;
    s0 = p0;
    two_sum(q0, p1, s1, s2);
    three_sum(s2, q1, p2);
    three_sum2(q1, q2, p3);
    s3 = q1;
    s4 = q2 + p2;
    return qd_renorm5_bf(s0, s1, s2, s3, s4);
}

// Fused s - a*b - c*d with ONE renormalisation (instead of two products and two sums,
// each renormalised).  Terms are collected by order (2^-53k of the operands' scale):
// order 0..2 products by TwoProd, order 3 plainly; each order is summed exactly with
// TwoSums whose errors drop to the next order; order 3 is summed plainly.  Error
// ~2^-208 of max(|s|, |ab|, |cd|) (tests/test_arith.py).
constexpr bool kQdLazy = true;
// Exact pairwise (tree) sum of N doubles: the rounded total, and the N - 1 TwoSum errors
// in a fixed order.  ceil(log2 N) dependent TwoSums instead of N - 1 for a running sum --
// the QD kernel runs one warp per SM sub-partition, so its time is these chains.
template <int N>
TOR_HD double tree_sum(const double (&t)[N], double* err) {
    if constexpr (N == 1) {
        return t[0];
    } else {
        constexpr int H = N / 2;
        double u[N - H];
        TOR_UNROLL
        for (int i = 0; i < H; ++i) two_sum(t[2 * i], t[2 * i + 1], u[i], err[i]);
        if constexpr (N & 1) u[H] = t[N - 1];
        return tree_sum<N - H>(u, err + H);
    }
}
// plain pairwise sum (the last order: its rounding errors are below the QD budget)
template <int N>
TOR_HD double tree_add(const double (&t)[N]) {
    if constexpr (N == 1) {
        return t[0];
    } else {
        constexpr int H = N / 2;
        double u[N - H];
        TOR_UNROLL
        for (int i = 0; i < H; ++i) u[i] = t[2 * i] + t[2 * i + 1];
        if constexpr (N & 1) u[H] = t[N - 1];
        return tree_add<N - H>(u);
    }
}
#define TOR_HD_R2 TOR_HD_RNI
template <bool kNorm>
TOR_HD qd qd_rank2_body(const qd& s, const qd& a, const qd& b, const qd& c, const qd& d) {
    double p0, e0, q0, f0;
    two_prod(a.x[0], b.x[0], p0, e0);
    two_prod(c.x[0], d.x[0], q0, f0);
    double pa, ea, pb, eb, qa, fa, qb, fb;
    two_prod(a.x[0], b.x[1], pa, ea);
    two_prod(a.x[1], b.x[0], pb, eb);
    two_prod(c.x[0], d.x[1], qa, fa);
    two_prod(c.x[1], d.x[0], qb, fb);
    double r[6], re[6];
    two_prod(a.x[0], b.x[2], r[0], re[0]);
    two_prod(a.x[1], b.x[1], r[1], re[1]);
    two_prod(a.x[2], b.x[0], r[2], re[2]);
    two_prod(c.x[0], d.x[2], r[3], re[3]);
    two_prod(c.x[1], d.x[1], r[4], re[4]);
    two_prod(c.x[2], d.x[0], r[5], re[5]);
    // order 0
    const double t0[3] = {s.x[0], -p0, -q0};
    double l1[2];
    const double h0 = tree_sum(t0, l1);
    // order 1
    const double t1[9] = {s.x[1], l1[0], l1[1], -e0, -f0, -pa, -pb, -qa, -qb};
    double l2[8];
    const double h1 = tree_sum(t1, l2);
    // order 2
    const double t2[19] = {s.x[2], l2[0], l2[1], l2[2], l2[3], l2[4], l2[5], l2[6], l2[7], -ea, -eb, -fa, -fb,
                           -r[0],  -r[1], -r[2], -r[3], -r[4], -r[5]};
    double l3[18];
    const double h2 = tree_sum(t2, l3);
    // order 3: plain
    const double t3[28] = {s.x[3], l3[0], l3[1], l3[2], l3[3], l3[4], l3[5], l3[6], l3[7], l3[8],
                           l3[9],  l3[10], l3[11], l3[12], l3[13], l3[14], l3[15], l3[16], l3[17],
                           -re[0], -re[1], -re[2], -re[3], -re[4], -re[5],
                           -fma_(a.x[0], b.x[3], a.x[1] * b.x[2]), -fma_(a.x[2], b.x[1], a.x[3] * b.x[0]),
                           -fma_(c.x[0], d.x[3], fma_(c.x[1], d.x[2], fma_(c.x[2], d.x[1], c.x[3] * d.x[0])))};
    const double h3 = tree_add(t3);
    if constexpr (kNorm) return qd_renorm5_bf(h0, h1, h2, h3, 0.0);
    else return qd{{h0, h1, h2, h3}};
}
template <bool kNorm>
TOR_HD_R2 qd qd_rank2_fused(qd s, qd a, qd b, qd c, qd d) {
    return qd_rank2_body<kNorm>(s, a, b, c, d);
}
// s - a*b, same scheme
template <bool kNorm>
TOR_HD qd qd_rank1_body(const qd& s, const qd& a, const qd& b) {
    double p0, e0, pa, ea, pb, eb, r[3], re[3];
    two_prod(a.x[0], b.x[0], p0, e0);
    two_prod(a.x[0], b.x[1], pa, ea);
    two_prod(a.x[1], b.x[0], pb, eb);
    two_prod(a.x[0], b.x[2], r[0], re[0]);
    two_prod(a.x[1], b.x[1], r[1], re[1]);
    two_prod(a.x[2], b.x[0], r[2], re[2]);
    const double t0[2] = {s.x[0], -p0};
    double l1[1];
    const double h0 = tree_sum(t0, l1);
    const double t1[5] = {s.x[1], l1[0], -e0, -pa, -pb};
    double l2[4];
    const double h1 = tree_sum(t1, l2);
    const double t2[10] = {s.x[2], l2[0], l2[1], l2[2], l2[3], -ea, -eb, -r[0], -r[1], -r[2]};
    double l3[9];
    const double h2 = tree_sum(t2, l3);
    const double t3[14] = {s.x[3], l3[0], l3[1], l3[2], l3[3], l3[4], l3[5], l3[6], l3[7], l3[8],
                           -re[0], -re[1], -re[2],
                           -fma_(a.x[0], b.x[3], fma_(a.x[1], b.x[2], fma_(a.x[2], b.x[1], a.x[3] * b.x[0])))};
    const double h3 = tree_add(t3);
    if constexpr (kNorm) return qd_renorm5_bf(h0, h1, h2, h3, 0.0);
    else return qd{{h0, h1, h2, h3}};
}
// a*b by the same order-collected scheme (products have no cancellation: without the
// final renormalisation the words are still ordered 2^-53k relative to |ab|)
template <bool kNorm>
TOR_HD_RNI qd qd_rank1_fused(qd s, qd a, qd b) {
    return qd_rank1_body<kNorm>(s, a, b);
}
template <bool kNorm>
TOR_HD qd qd_mul_body(const qd& a, const qd& b) {
    double p0, e0, pa, ea, pb, eb, r[3], re[3];
    two_prod(a.x[0], b.x[0], p0, e0);
    two_prod(a.x[0], b.x[1], pa, ea);
    two_prod(a.x[1], b.x[0], pb, eb);
    two_prod(a.x[0], b.x[2], r[0], re[0]);
    two_prod(a.x[1], b.x[1], r[1], re[1]);
    two_prod(a.x[2], b.x[0], r[2], re[2]);
    const double t1[3] = {e0, pa, pb};
    double l2[2];
    const double h1 = tree_sum(t1, l2);
    const double t2[7] = {r[0], r[1], r[2], ea, eb, l2[0], l2[1]};
    double l3[6];
    const double h2 = tree_sum(t2, l3);
    const double t3[10] = {re[0], re[1], re[2], l3[0], l3[1], l3[2], l3[3], l3[4], l3[5],
                           fma_(a.x[0], b.x[3], fma_(a.x[1], b.x[2], fma_(a.x[2], b.x[1], a.x[3] * b.x[0])))};
    const double h3 = tree_add(t3);
    if constexpr (kNorm) return qd_renorm_lead(p0, h1, h2, h3);
    else return qd{{p0, h1, h2, h3}};
}
template <bool kNorm>
TOR_HD_RNI qd qd_mul_fused(qd a, qd b) {
    return qd_mul_body<kNorm>(a, b);
}

// Schur-state updates skip the final renormalisation (like the lazy DD products): every
// state entry is O(1) in absolute terms (|S_ij| <= max_k R_kk), so words ordered by
// ABSOLUTE scale 2^-53k keep the fused algorithm's error at ~2^-208 of that scale even
// when the leading word has cancelled; entries are renormalised where they become
// pivots, and the products that consume them renormalise their results.
// (thin inline wrappers: one out-of-line call per update, to the fused body)
TOR_HD qd qd_rank2(const qd& s, const qd& a, const qd& b, const qd& c, const qd& d) {
    return qd_rank2_fused<!kQdLazy>(s, a, b, c, d);
}
TOR_HD qd qd_rank1(const qd& s, const qd& a, const qd& b) { return qd_rank1_fused<true>(s, a, b); }
TOR_HD qd qd_rank1_lazy(const qd& s, const qd& a, const qd& b) { return qd_rank1_fused<!kQdLazy>(s, a, b); }

// 1/sqrt(x), x > 0 normalised: DD value y = (y0, y1) (~2^-104), then one Newton step
// y + y e / 2 with e = 1 - x y^2 by the fused rank-1 (y^2 formed exactly enough from
// TwoProds of the DD words) and the correction as a DD product (e ~ 2^-104 needs only
// ~2^-106 relative).  One renormalisation.
// kInl: the residual's fused rank-1 inline (inside the out-of-line QD pivot / leaf) or as
// its one out-of-line copy
template <bool kInl>
TOR_HD qd qd_rsqrt_body(const qd& x) {
    const dd y = dd_rsqrt(dd_norm(dd{x.x[0], x.x[1]}));
    // y^2 = p + (pe + q) + (qe + ll) + lle, words by order (2^-53k)
    double p, pe, q, qe, ll, lle, m1, m2, n2, n3, n4;
    two_prod(y.hi, y.hi, p, pe);
    two_prod(2.0 * y.hi, y.lo, q, qe);
    two_prod(y.lo, y.lo, ll, lle);
    two_sum(pe, q, m1, m2);
    two_sum(m2, qe, n2, n3);
    two_sum(n2, ll, n2, n4);
    const qd y2{{p, m1, n2, (n3 + n4) + lle}};
    const qd one{{1.0, 0.0, 0.0, 0.0}};
    qd e;
    if constexpr (kInl) e = qd_rank1_body<true>(one, x, y2);
    else e = qd_rank1_fused<true>(one, x, y2);
    // corr = (y/2) * (e0 + e1), DD product
    double c0, c1;
    two_prod(0.5 * y.hi, e.x[0], c0, c1);
    c1 = fma_(0.5 * y.hi, e.x[1], c1);
    c1 = fma_(0.5 * y.lo, e.x[0], c1);
    return qd_renorm_lead(y.hi, y.lo, c0, c1);
}
TOR_HD_NI qd qd_rsqrt_fast(qd x) { return qd_rsqrt_body<false>(x); }
// 1/sqrt(x), x > 0: DD seed then one QD Newton step y + y(1 - x y^2)/2.
TOR_HD_NI qd qd_rsqrt_slow(qd x) {
    const dd ys = dd_rsqrt(dd_norm(dd{x.x[0], x.x[1]}));
    const qd y = qd{{ys.hi, ys.lo, 0.0, 0.0}};
    const qd y2 = qd_mul(y, y);
    const qd xy2 = qd_mul(x, y2);
    const qd r = qd_sub(qd_make(1.0), xy2);  // ~2^-104
    const qd corr = qd_mul(y, qd_mul_d(r, 0.5));
    return qd_add(y, corr);
}

TOR_HD qd qd_rsqrt(const qd& x) { return qd_rsqrt_fast(x); }

// ================================================================ traits ==
// Uniform interface used by the kernels.  Word type W, number of doubles K.
template <class T> struct Arith;

template <> struct Arith<double> {
    static constexpr int K = 1;
    TOR_HD static double zero() { return 0.0; }
    TOR_HD static double one() { return 1.0; }
    TOR_HD static double from(double x) { return x; }
    TOR_HD static double hi(double a) { return a; }
    TOR_HD static double norm(double a) { return a; }
    // a double with the sign of the (possibly unnormalised) value: for sign tests
    TOR_HD static double sign_val(double a) { return a; }
    TOR_HD static double mul(double a, double b) { return a * b; }
    TOR_HD static double rank2(double s, double a, double b, double c, double d) {
        return fma_(-c, d, fma_(-a, b, s));
    }
    TOR_HD static double rank1(double s, double a, double b) { return fma_(-a, b, s); }
    TOR_HD static double rank2_item(double s, double a, double b, double c, double d) { return rank2(s, a, b, c, d); }
    TOR_HD static double rank1s(double s, double a, double b) { return fma_(-a, b, s); }
    TOR_HD static double rsqrt(double a) { return rsqrt_d(a); }
    TOR_HD static double unb(double a) { return a; }
    // pivot-row vector pair: u = s0 r1, w = (s1 - u1 u) r2 (s0, s1 state entries; u, w may alias them)
    TOR_HD static void vec(double s0, double s1, double r1, double u1, double r2, double& u, double& w) {
        const double uu = s0 * r1;
        w = fma_(-u1, uu, s1) * r2;
        u = uu;
    }
    TOR_HD static double neg(double a) { return -a; }
    TOR_HD static void words(double a, double* w) { w[0] = a; }
};

template <> struct Arith<dd> {
    static constexpr int K = 2;
    TOR_HD static dd zero() { return dd{0.0, 0.0}; }
    TOR_HD static dd one() { return dd{1.0, 0.0}; }
    TOR_HD static dd from(double x) { return dd{x, 0.0}; }
    TOR_HD static double hi(const dd& a) { return a.hi; }
    TOR_HD static dd norm(const dd& a) { return dd_norm(a); }
    TOR_HD static double sign_val(const dd& a) { return a.hi + a.lo; }
    // Products feed further products, rank updates or the accumulator, all of which use
    // both words: the final renormalisation is skipped (|lo| <= 2 ulp(hi)); values are
    // renormalised explicitly where it matters (pivots before rsqrt).
    TOR_HD static dd mul(const dd& a, const dd& b) {
        double p, e;
        two_prod(a.hi, b.hi, p, e);
        e = fma_(a.hi, b.lo, e);
        e = fma_(a.lo, b.hi, e);
        return dd{p, e};
    }
    static constexpr bool kGrid = true;
    // Schur-state updates: fixed-exponent (grid) DD
    TOR_HD static dd rank2(const dd& s, const dd& a, const dd& b, const dd& c, const dd& d) {
        return dd_rank2_grid(s, a, b, c, d);
    }
    TOR_HD static dd rank1s(const dd& s, const dd& a, const dd& b) { return dd_rank1_grid(s, a, b); }
    // state entry -> value
    TOR_HD static dd unb(const dd& a) { return dd_unbias(a); }
    TOR_HD static void vec(const dd& s0, const dd& s1, const dd& r1, const dd& u1, const dd& r2, dd& u, dd& w) {
        const dd uu = mul(unb(s0), r1);
        w = mul(rank1s(s1, u1, uu), r2);
        u = uu;
    }
    // general (non-state) s - a*b
    TOR_HD static dd rank1(const dd& s, const dd& a, const dd& b) { return dd_rank1(s, a, b); }
    TOR_HD static dd rank2_item(const dd& s, const dd& a, const dd& b, const dd& c, const dd& d) {
        return rank2(s, a, b, c, d);
    }
    TOR_HD static dd rsqrt(const dd& a) { return dd_rsqrt(a); }
    TOR_HD static dd neg(const dd& a) { return dd_neg(a); }
    TOR_HD static void words(const dd& a, double* w) {
        w[0] = a.hi;
        w[1] = a.lo;
    }
};

template <> struct Arith<qd> {
    static constexpr int K = 4;
    TOR_HD static qd zero() { return qd{{0.0, 0.0, 0.0, 0.0}}; }
    TOR_HD static qd one() { return qd{{1.0, 0.0, 0.0, 0.0}}; }
    TOR_HD static qd from(double x) { return qd{{x, 0.0, 0.0, 0.0}}; }
    TOR_HD static double hi(const qd& a) { return a.x[0]; }
    TOR_HD static qd norm(const qd& a) { return qd_renorm5_bf(a.x[0], a.x[1], a.x[2], a.x[3], 0.0); }
    TOR_HD static double sign_val(const qd& a) { return (a.x[0] + a.x[1]) + (a.x[2] + a.x[3]); }
    TOR_HD static qd mul(const qd& a, const qd& b) { return qd_mul_fused<true>(a, b); }
    TOR_HD static qd rank2(const qd& s, const qd& a, const qd& b, const qd& c, const qd& d) {
        return qd_rank2(s, a, b, c, d);
    }
    TOR_HD static qd rank2_item(const qd& s, const qd& a, const qd& b, const qd& c, const qd& d) {
        return rank2(s, a, b, c, d);
    }
    TOR_HD static qd rank1(const qd& s, const qd& a, const qd& b) { return qd_rank1(s, a, b); }
    TOR_HD static qd rank1s(const qd& s, const qd& a, const qd& b) { return qd_rank1_lazy(s, a, b); }
    TOR_HD static qd rsqrt(const qd& a) { return qd_rsqrt(a); }
    // a*c - b*b (2x2 determinant) by one fused update
    TOR_HD static qd det2(const qd& a, const qd& b, const qd& c) {
        return qd_rank2_fused<true>(qd{{0.0, 0.0, 0.0, 0.0}}, qd_neg(a), c, b, b);
    }
    TOR_HD static qd unb(const qd& a) { return a; }
    TOR_HD static void vec(const qd& s0, const qd& s1, const qd& r1, const qd& u1, const qd& r2, qd& u, qd& w);
    TOR_HD static qd neg(const qd& a) { return qd_neg(a); }
    TOR_HD static void words(const qd& a, double* w) {
        for (int i = 0; i < 4; ++i) w[i] = a.x[i];
    }
};

// ============================================================= pivots ==
// Pivot chain of one mode elimination (rows 0,1 of the view): Cholesky pivots
// rho1 = 1/sqrt(s00) and rho2 = 1/sqrt(s11 - s01^2/s00), computed as
// rho2 = sqrt(s00) * rhod with rhod = 1/sqrt(det2), det2 = s00 s11 - s01^2, so the
// two reciprocal square roots are independent (half the dependent latency of the
// textbook chain); the child's term factor is t * rhod.  s00, s01, s11 are state
// entries (biased in grid DD).
template <class T> struct Piv {
    T r1, u1, r2, tn;
    bool bad0, bad1;
};
template <class T>
TOR_HD Piv<T> pivot2(const T& s00, const T& s01, const T& s11, const T& t) {
    using A = Arith<T>;
    Piv<T> p;
    const T a = A::norm(A::unb(s00));
    const T b01 = A::unb(s01);
    p.bad0 = nonpositive(A::hi(a));
    p.r1 = A::rsqrt(a);
    const T det = A::norm(A::rank1(A::mul(a, A::unb(s11)), b01, b01));
    p.bad1 = nonpositive(A::hi(det));
    const T rd = A::rsqrt(det);
    p.u1 = A::mul(b01, p.r1);
    p.r2 = A::mul(A::mul(a, p.r1), rd);
    p.tn = A::mul(t, rd);
    return p;
}

// DD: the two reciprocal square roots start from seeds of the un-normalised leading
// words (MUFU latency overlaps the renormalisations), det by dd_det2 (one TwoSum).
template <>
TOR_HD Piv<dd> pivot2<dd>(const dd& s00, const dd& s01, const dd& s11, const dd& t) {
    using A = Arith<dd>;
    Piv<dd> p;
    const dd a0 = A::unb(s00), b = A::unb(s01), c = A::unb(s11);
    const double y1 = rsqrt_seed(a0.hi);
    const dd a = dd_norm(a0);
    p.bad0 = nonpositive(a.hi);
    double h;
    const dd det = dd_det2(a0, b, c, h);
    const double yd = rsqrt_seed(h);
    p.bad1 = nonpositive(det.hi);
    p.r1 = dd_rsqrt_seeded(a, y1);
    const dd rd = dd_rsqrt_seeded(det, yd);
    p.u1 = A::mul(b, p.r1);
    p.r2 = A::mul(A::mul(a, p.r1), rd);
    p.tn = A::mul(t, rd);
    return p;
}
// QD: det by one fused update
// (one out-of-line body per pivot with its products, determinant and reciprocal square
// roots inline: one call instead of ~8, and the two rsqrt chains schedule together)
TOR_HD_RNI Piv<qd> qd_pivot_ool(qd s00, qd s01, qd s11, qd t) {
    Piv<qd> p;
    const qd a = qd_renorm5_bf(s00.x[0], s00.x[1], s00.x[2], s00.x[3], 0.0);
    p.bad0 = nonpositive(a.x[0]);
    p.r1 = qd_rsqrt_body<true>(a);
    const qd det = qd_rank2_body<true>(qd{{0.0, 0.0, 0.0, 0.0}}, qd_neg(a), s11, s01, s01);
    p.bad1 = nonpositive(det.x[0]);
    const qd rd = qd_rsqrt_body<true>(det);
    p.u1 = qd_mul_body<true>(s01, p.r1);
    p.r2 = qd_mul_body<true>(qd_mul_body<true>(a, p.r1), rd);
    p.tn = qd_mul_body<true>(t, rd);
    return p;
}
template <>
TOR_HD Piv<qd> pivot2<qd>(const qd& s00, const qd& s01, const qd& s11, const qd& t) {
    return qd_pivot_ool(s00, s01, s11, t);
}
#if defined(__CUDA_ARCH__)
// The same pivot for lanes that share it (the warp-cooperative fan-out levels and DFS steps
// compute one pivot in >= 2 lanes): the lane with role 0 runs the reciprocal square root of
// s00 and the products with it (u1, s00 rho1), its partner lane ^ xm (role 1, same inputs)
// that of the determinant and t rhod, then they exchange -- one rsqrt and three products per
// lane instead of two and four (QD: ~780 instead of ~1090 FP64 instructions per pivot; the
// same bodies on the same operands, so every value is bit-identical to qd_pivot_ool).
__device__ __noinline__ Piv<qd> qd_pivot_split_ool(qd s00, qd s01, qd s11, qd t, bool role, int xm) {
    Piv<qd> p;
    const qd a = qd_renorm5_bf(s00.x[0], s00.x[1], s00.x[2], s00.x[3], 0.0);
    p.bad0 = nonpositive(a.x[0]);
    const qd det = qd_rank2_body<true>(qd{{0.0, 0.0, 0.0, 0.0}}, qd_neg(a), s11, s01, s01);
    p.bad1 = nonpositive(det.x[0]);
    qd x, f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        x.x[i] = role ? det.x[i] : a.x[i];
        f.x[i] = role ? t.x[i] : s01.x[i];
    }
    const qd y = qd_rsqrt_body<true>(x);     // rho1 | rhod
    const qd m1 = qd_mul_body<true>(f, y);   // u1 = s01 rho1 | tn = t rhod
    const qd m2 = qd_mul_body<true>(a, y);   // s00 rho1 | (unused)
    qd ar, rd;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double yo = __shfl_xor_sync(0xffffffffu, y.x[i], xm);
        const double m1o = __shfl_xor_sync(0xffffffffu, m1.x[i], xm);
        const double m2o = __shfl_xor_sync(0xffffffffu, m2.x[i], xm);
        p.r1.x[i] = role ? yo : y.x[i];
        rd.x[i] = role ? y.x[i] : yo;
        p.u1.x[i] = role ? m1o : m1.x[i];
        p.tn.x[i] = role ? m1.x[i] : m1o;
        ar.x[i] = role ? m2o : m2.x[i];
    }
    p.r2 = qd_mul_body<true>(ar, rd);
    return p;
}
#endif
// Pivot shared by the lanes l and l ^ xm (all 32 lanes call it): the split form for QD, the
// plain pivot otherwise
template <class T>
TOR_HD Piv<T> pivot2_shared(const T& s00, const T& s01, const T& s11, const T& t, int lane, int xm) {
    (void)lane;
    (void)xm;
    return pivot2<T>(s00, s01, s11, t);
}
#if defined(__CUDA_ARCH__)
template <>
__device__ __forceinline__ Piv<qd> pivot2_shared<qd>(const qd& s00, const qd& s01, const qd& s11, const qd& t,
                                                       int lane, int xm) {
    return qd_pivot_split_ool(s00, s01, s11, t, (lane & xm) != 0, xm);
}
#endif
// QD pivot-row vector pair in one out-of-line body (one call instead of three)
struct QdPair {
    qd u, w;
};
TOR_HD_RNI QdPair qd_vec_ool(qd s0, qd s1, qd r1, qd u1, qd r2) {
    const qd u = qd_mul_body<true>(s0, r1);
    return QdPair{u, qd_mul_body<true>(qd_rank1_body<!kQdLazy>(s1, u1, u), r2)};
}
TOR_HD void Arith<qd>::vec(const qd& s0, const qd& s1, const qd& r1, const qd& u1, const qd& r2, qd& u, qd& w) {
    const QdPair p = qd_vec_ool(s0, s1, r1, u1, r2);
    u = p.u;
    w = p.w;
}
// Term factor of a one-mode (leaf) state: t / sqrt(det).
template <class T>
TOR_HD T leaf_term(const T& s00, const T& s01, const T& s11, const T& t, bool& bad) {
    using A = Arith<T>;
    const T b = A::unb(s01);
    const T det = A::norm(A::rank1(A::mul(A::unb(s00), A::unb(s11)), b, b));
    bad = nonpositive(A::hi(det));
    return A::mul(t, A::rsqrt(det));
}
struct QdLeaf {
    qd v;
    bool bad;
};
TOR_HD_RNI QdLeaf qd_leaf_ool(qd s00, qd s01, qd s11, qd t) {
    const qd det = qd_rank2_body<true>(qd{{0.0, 0.0, 0.0, 0.0}}, qd_neg(s00), s11, s01, s01);
    return QdLeaf{qd_mul_body<true>(t, qd_rsqrt_body<true>(det)), nonpositive(det.x[0])};
}
template <>
TOR_HD qd leaf_term<qd>(const qd& s00, const qd& s01, const qd& s11, const qd& t, bool& bad) {
    const QdLeaf r = qd_leaf_ool(s00, s01, s11, t);
    bad = r.bad;
    return r.v;
}
template <>
TOR_HD dd leaf_term<dd>(const dd& s00, const dd& s01, const dd& s11, const dd& t, bool& bad) {
    using A = Arith<dd>;
    double h;
    const dd det = dd_det2(A::unb(s00), A::unb(s01), A::unb(s11), h);
    bad = nonpositive(det.hi);
    return A::mul(t, dd_rsqrt_seeded(det, rsqrt_seed(h)));
}

// ========================================================== accumulators ==
// Signed term accumulation.  fp64 and DD terms accumulate in an accurate DD sum,
// QD terms in QD.  Sum |t| is carried in fp64 for the posterior cancellation check.
// kScaled: the input was scaled by 2^-sc (DD grid states need max R_kk < 3.75; physical
// states have R_kk <= 2 and never are), so each term is multiplied back by 2^(sc |Z|).  A
// compile-time switch: a runtime `if (sc)` is if-converted and costs every term.
template <class T, bool kScaled = false> struct Acc;

// x or -x: one integer XOR of the sign bit (no select on both words)
TOR_HD double flip_sign(double x, bool negative) {
#if defined(__CUDA_ARCH__)
    return __hiloint2double(__double2hiint(x) ^ (static_cast<int>(negative) << 31), __double2loint(x));
#else
    return negative ? -x : x;
#endif
}

// term scaling for scaled inputs (R -> 2^-s R multiplies t(Z) by 2^(s|Z|)): exact
TOR_HD double pow2i(int e) {
#if defined(__CUDA_ARCH__)
    return __hiloint2double((1023 + e) << 20, 0);
#else
    return std::ldexp(1.0, e);
#endif
}

template <bool kScaled> struct Acc<double, kScaled> {
    dd s{0.0, 0.0};
    double abs_sum = 0.0;
    int sc = 0;
    TOR_HD void add(double t, bool negative, int z) {
        if constexpr (kScaled) t *= pow2i(-sc * z);
        const double v = flip_sign(t, negative);
        double h, e;
        two_sum(s.hi, v, h, e);
        s.hi = h;
        s.lo += e;
        abs_sum += fabs(t);
    }
    TOR_HD void flush() {}
    TOR_HD void merge(const Acc& o) {
        s = dd_add(s, o.s);
        abs_sum += o.abs_sum;
    }
    TOR_HD void words(double* w) const {
        const dd n = dd_norm(s);
        w[0] = n.hi;
        w[1] = n.lo;
        w[2] = 0.0;
        w[3] = 0.0;
    }
};

template <bool kScaled> struct Acc<dd, kScaled> {
    // running sum s (accurate DD) + a lazily renormalised block (h, c): per term one
    // TwoSum on the leading words and one plain add for the low words; the block is
    // folded into s by flush() every few terms (lane subtrees), keeping the lazy
    // error below 2^-98 of the block's term magnitudes.
    dd s{0.0, 0.0};
    double h = 0.0, c = 0.0;
    double abs_sum = 0.0;
    int sc = 0;
    TOR_HD void add(dd t, bool negative, int z) {
        if constexpr (kScaled) {
            const double f = pow2i(-sc * z);
            t.hi *= f;
            t.lo *= f;
        }
        const double th = flip_sign(t.hi, negative);  // 85.7 vs 86.2 ms with selects (n=32)
        const double tl = flip_sign(t.lo, negative);
        double nh, e;
        two_sum(h, th, nh, e);
        h = nh;
        c += tl + e;
        abs_sum += fabs(t.hi);
    }
    TOR_HD void flush() {
        s = dd_add(s, dd_norm(dd{h, c}));
        h = 0.0;
        c = 0.0;
    }
    TOR_HD void merge(const Acc& o) {
        s = dd_add(s, o.s);
        abs_sum += o.abs_sum;
    }
    TOR_HD void words(double* w) const {
        w[0] = s.hi;
        w[1] = s.lo;
        w[2] = 0.0;
        w[3] = 0.0;
    }
};

template <bool kScaled> struct Acc<qd, kScaled> {
    // running sum s (renormalised QD) + a lazy block b: per term, exact TwoSums on the
    // words of orders 0..2 (each order's errors into the next order), order 3 plainly;
    // the block is renormalised and added to s by flush() (every lane subtree).
    qd s{{0.0, 0.0, 0.0, 0.0}};
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
    double abs_sum = 0.0;
    int sc = 0;
    TOR_HD void add(const qd& t, bool negative, int z) {
        (void)z;  // QD words are never grid-scaled
        double e0, e1, e2, e3, e4, e5;
        two_sum(b0, flip_sign(t.x[0], negative), b0, e0);
        two_sum(b1, flip_sign(t.x[1], negative), b1, e1);
        two_sum(b1, e0, b1, e2);
        two_sum(b2, flip_sign(t.x[2], negative), b2, e3);
        two_sum(b2, e1, b2, e4);
        two_sum(b2, e2, b2, e5);
        b3 += ((flip_sign(t.x[3], negative) + e3) + e4) + e5;
        abs_sum += fabs(t.x[0]);
    }
    TOR_HD void flush() {
        s = qd_add(s, qd_renorm5_bf(b0, b1, b2, b3, 0.0));
        b0 = b1 = b2 = b3 = 0.0;
    }
    TOR_HD void merge(const Acc& o) {
        s = qd_add(s, o.s);
        abs_sum += o.abs_sum;
    }
    TOR_HD void words(double* w) const {
        for (int i = 0; i < 4; ++i) w[i] = s.x[i];
    }
};

}  // namespace tor
