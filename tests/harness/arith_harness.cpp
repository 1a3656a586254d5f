// Host build of the engine's multi-word arithmetic (paper_2009_01177_b200/csrc/arith.cuh,
// the same source the kernels compile) for exact-rational unit tests (tests/test_arith.py).
// Built by the test with g++ -O2 -ffp-contract=off, loaded through ctypes.  Arrays are
// words in order (DD: hi, lo; QD: x0..x3).
#include "../../paper_2009_01177_b200/csrc/arith.cuh"

using namespace tor;

static dd D(const double* p) { return dd{p[0], p[1]}; }
static qd Q(const double* p) { return qd{{p[0], p[1], p[2], p[3]}}; }
static void put(const dd& v, double* o) { o[0] = v.hi; o[1] = v.lo; }
static void put(const qd& v, double* o) { for (int i = 0; i < 4; ++i) o[i] = v.x[i]; }

extern "C" {
double h_grid_c() { return kGridC; }
void h_dd_to_grid(double x, double y, double* o) { put(dd_to_grid(x, y), o); }
void h_dd_rank2(const double* s, const double* a, const double* b, const double* c, const double* d, double* o) {
    put(Arith<dd>::rank2(D(s), D(a), D(b), D(c), D(d)), o);
}
void h_dd_rank1s(const double* s, const double* a, const double* b, double* o) {
    put(Arith<dd>::rank1s(D(s), D(a), D(b)), o);
}
void h_dd_mul(const double* a, const double* b, double* o) { put(Arith<dd>::mul(D(a), D(b)), o); }
void h_dd_rsqrt(const double* x, double* o) { put(dd_rsqrt(D(x)), o); }
void h_dd_det2(const double* a, const double* b, const double* c, double* o) {
    double h;
    put(dd_det2(D(a), D(b), D(c), h), o);
}
// pivots of biased state entries: out = r1, u1, r2, tn (2 words each), flags
int h_dd_pivot(const double* s00, const double* s01, const double* s11, const double* t, double* o) {
    const Piv<dd> p = pivot2<dd>(D(s00), D(s01), D(s11), D(t));
    put(p.r1, o);
    put(p.u1, o + 2);
    put(p.r2, o + 4);
    put(p.tn, o + 6);
    return (p.bad0 ? 1 : 0) | (p.bad1 ? 2 : 0);
}
int h_dd_leaf(const double* s00, const double* s01, const double* s11, const double* t, double* o) {
    bool bad;
    put(leaf_term<dd>(D(s00), D(s01), D(s11), D(t), bad), o);
    return bad ? 1 : 0;
}
void h_qd_add(const double* a, const double* b, double* o) { put(qd_add(Q(a), Q(b)), o); }
void h_qd_mul(const double* a, const double* b, double* o) { put(qd_mul(Q(a), Q(b)), o); }
void h_qd_rank2(const double* s, const double* a, const double* b, const double* c, const double* d, double* o) {
    put(Arith<qd>::rank2(Q(s), Q(a), Q(b), Q(c), Q(d)), o);
}
void h_qd_rsqrt(const double* x, double* o) { put(qd_rsqrt(Q(x)), o); }
int h_qd_pivot(const double* s00, const double* s01, const double* s11, const double* t, double* o) {
    const Piv<qd> p = pivot2<qd>(Q(s00), Q(s01), Q(s11), Q(t));
    put(p.r1, o);
    put(p.u1, o + 4);
    put(p.r2, o + 8);
    put(p.tn, o + 12);
    return (p.bad0 ? 1 : 0) | (p.bad1 ? 2 : 0);
}
// DD accumulator: adds n terms (2 words each) with signs, flushing every `flush` terms
void h_dd_acc(const double* t, const int* neg, int n, int flush, double* o) {
    Acc<dd> a;
    for (int i = 0; i < n; ++i) {
        a.add(D(t + 2 * i), neg[i] != 0, 0);
        if (flush && (i + 1) % flush == 0) a.flush();
    }
    a.flush();
    double w[4];
    a.words(w);
    o[0] = w[0];
    o[1] = w[1];
    o[2] = a.abs_sum;
}
}
extern "C" void h_qd_mul_fused(const double* a, const double* b, double* o) {
    put(Arith<qd>::mul(Q(a), Q(b)), o);
}
// QD accumulator: n terms (4 words each), flush every `flush` terms; out = 4 words, sum|t|
extern "C" void h_qd_acc(const double* t, const int* neg, int n, int flush, double* o) {
    Acc<qd> a;
    for (int i = 0; i < n; ++i) {
        a.add(Q(t + 4 * i), neg[i] != 0, 0);
        if (flush && (i + 1) % flush == 0) a.flush();
    }
    a.flush();
    double w[4];
    a.words(w);
    for (int i = 0; i < 4; ++i) o[i] = w[i];
    o[4] = a.abs_sum;
}
extern "C" void h_qd_vec(const double* s0, const double* s1, const double* r1, const double* u1,
                         const double* r2, double* u, double* w) {
    qd uu, ww;
    Arith<qd>::vec(Q(s0), Q(s1), Q(r1), Q(u1), Q(r2), uu, ww);
    put(uu, u);
    put(ww, w);
}
