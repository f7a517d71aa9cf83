// The 15-feature triangle-pair distance over shared-memory-staged triangles.
//
// Same arithmetic as geom.cuh's feature_dist (bit-identical results), laid
// out for FP64 throughput on sm_100a:
//  * the two world triangles, their edge vectors and squared edge lengths are
//    staged once per row in shared memory, structure-of-arrays across the
//    block (element k of thread t at s[k * kStride + t]: conflict-free, and
//    with a compile-time stride every access is an immediate-offset LDS);
//  * the six point-triangle and nine segment-segment features run as two
//    compact loops -- one copy of each feature's code stays in the
//    instruction cache;
//  * each feature is branch-free: the Voronoi region (point-triangle) and the
//    clamp case (segment-segment) only select operands, and every lane runs
//    the same instruction stream; divisions are predicated on the lanes that
//    need them;
//  * divisions are skipped wherever their rounded quotient cannot matter:
//    np.clip(num / den, 0, 1) with den > 0 is exactly 0 for num <= 0 and
//    exactly 1 for num >= den; t > 1 is decided exactly without dividing;
//  * comparisons against zero and the running minimum use integer compares
//    on the IEEE bit patterns (exact for the finite values that occur), which
//    keeps them off the FP64 pipe.
#pragma once

#include "geom.cuh"

namespace ltsg {

// Staged row layout (doubles): A corners 0..8, B corners 9..17, A edges
// 18..26, B edges 27..35, |eA|^2 36..38, |eB|^2 39..41.
constexpr int kStA = 0, kStB = 9, kStEA = 18, kStEB = 27, kStAA = 36, kStBB = 39;
constexpr int kStaged = 42;

template <int kStride>
struct Staged {
  double* s;
  __device__ __forceinline__ double& at(int k) const { return s[k * kStride]; }
  __device__ __forceinline__ V3 v3(int k) const { return V3{at(k), at(k + 1), at(k + 2)}; }
  __device__ __forceinline__ void put(int k, V3 v) const {
    at(k) = v.x;
    at(k + 1) = v.y;
    at(k + 2) = v.z;
  }
};

// Exact comparisons with zero through the bit pattern (finite x):
// x <= 0.0 holds for -0.0 (INT64_MIN) and every negative; x >= 0.0 for +0.0,
// -0.0 and every positive; x < 0.0 for negatives except -0.0.
#ifndef LTSG_SIGN_INT
#define LTSG_SIGN_INT 0
#endif
#if LTSG_SIGN_INT
__device__ __forceinline__ bool le0(double x) { return __double_as_longlong(x) <= 0; }
__device__ __forceinline__ bool ge0(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 || b == (long long)0x8000000000000000ULL;
}
__device__ __forceinline__ bool lt0(double x) {
  const long long b = __double_as_longlong(x);
  return b < 0 && b != (long long)0x8000000000000000ULL;
}
// min of two non-negative doubles (squared distances) by their bit patterns
__device__ __forceinline__ double min_nonneg(double a, double b) {
  const unsigned long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double(x < y ? x : y);
}
#else
// one DSETP each: the kernel is issue-bound, and a 64-bit integer compare
// costs two or three integer instructions
__device__ __forceinline__ bool le0(double x) { return x <= 0.0; }
__device__ __forceinline__ bool ge0(double x) { return x >= 0.0; }
__device__ __forceinline__ bool lt0(double x) { return x < 0.0; }
__device__ __forceinline__ double min_nonneg(double a, double b) { return b < a ? b : a; }
#endif

template <int kStride>
__device__ __forceinline__ void stage_pair(const Staged<kStride>& st, const Tri& a, const Tri& b) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    st.put(kStA + 3 * k, a.v[k]);
    st.put(kStB + 3 * k, b.v[k]);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const V3 ea = a.v[(k + 1) % 3] - a.v[k];
    const V3 eb = b.v[(k + 1) % 3] - b.v[k];
    st.put(kStEA + 3 * k, ea);
    st.put(kStEB + 3 * k, eb);
    st.at(kStAA + k) = dot_simd(ea, ea);
    st.at(kStBB + k) = dot_simd(eb, eb);
  }
}

// np.clip(num / den, 0, 1) for den > 1e-300 (so _safe_div divides by den):
// a non-positive numerator gives a quotient <= 0 (or -0) that clips to +0, a
// numerator >= den gives a quotient >= 1 that clips to 1, so only
// 0 < num < den divides.
__device__ __forceinline__ double clip_quot(double num, double den) {
  double q = 0.0;
  if (num > 0.0 && num < den) q = dv(num, den);
  else if (num >= den) q = 1.0;
  return q;
}

// Squared point-triangle distance (kernels.py:23-75), branch-free.
// ab = e0, ac = -e2 (exact negation of v0 - v2), bc = e1.  The closest point
// is q = (P + D1*s1) + ac*s2: vertex regions use s1 = s2 = 0 (q == P up to
// the sign of zeros, which squaring removes), edges s2 = 0.  P and D1 are
// re-read from the stage by index instead of being moved between registers.
template <int kStride>
__device__ __forceinline__ double pt_sq_staged(const Staged<kStride>& st, int pk, int tb, int eb) {
  const V3 p = st.v3(pk);
  const V3 a = st.v3(tb), b = st.v3(tb + 3), c = st.v3(tb + 6);
  const V3 ab = st.v3(eb), ac = neg(st.v3(eb + 6));
  const V3 ap = p - a, bp = p - b, cp = p - c;
  const double d1 = dot_simd(ab, ap), d2 = dot_simd(ac, ap);
  const double d3 = dot_simd(ab, bp), d4 = dot_simd(ac, bp);
  const double d5 = dot_simd(ab, cp), d6 = dot_simd(ac, cp);
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  const double vb = sub(mul(d5, d2), mul(d1, d6));
  const double va = sub(mul(d3, d6), mul(d5, d4));
  const double e43 = sub(d4, d3), e56 = sub(d5, d6);
  const bool in_a = le0(d1) && le0(d2);
  const bool in_b = ge0(d3) && d4 <= d3;
  const bool in_c = ge0(d6) && d5 <= d6;
  const bool on_ab = le0(vc) && ge0(d1) && le0(d3);
  const bool on_ac = le0(vb) && ge0(d2) && le0(d6);
  const bool on_bc = le0(va) && ge0(e43) && ge0(e56);
  const bool vertex = in_a || in_b || in_c;
  // region -> (vertex index of P, edge of D1, quotient); later overrides earlier
  const double den = add(add(va, vb), vc);
  int pv = 0, de = 0;  // P = a, D1 = ab
  double n1 = vb, m1 = den;
  bool face = true;
  if (on_bc) { n1 = e43; m1 = add(e43, e56); pv = 1; de = 1; face = false; }
  if (on_ac) { n1 = d2; m1 = sub(d2, d6); pv = 0; de = 2; face = false; }
  if (on_ab) { n1 = d1; m1 = sub(d1, d3); pv = 0; de = 0; face = false; }
  if (vertex) { pv = in_a ? 0 : (in_b ? 1 : 2); face = false; }
  double s1 = 0.0, s2 = 0.0;
  if (!vertex) s1 = sdiv(n1, m1);
  if (face) s2 = sdiv(vc, den);
  const V3 P = st.v3(tb + 3 * pv);
  V3 D1 = st.v3(eb + 3 * de);
  if (de == 2) D1 = neg(D1);
  const V3 q = (P + scale(D1, s1)) + scale(ac, s2);
  return sqn(p - q);
}

// Squared distance of segments [p1, p1+u], [p2, p2+w] (kernels.py:78-115),
// branch-free; uu = |u|^2, ww = |w|^2 (dot_simd order).
__device__ __forceinline__ double ss_sq_uniform(V3 p1, V3 u, double uu, V3 p2, V3 w, double ww) {
  if (!(uu > 1e-280) || !(ww > 1e-280)) return segment_segment_sq<false>(p1, u, uu, p2, w, ww);
  const V3 r = p1 - p2;
  const double wr = dot_simd(w, r);
  const double ur = dot_simd(u, r);
  const double uw = dot_simd(u, w);
  const double det = sub(mul(uu, ww), mul(uw, uw));
  // parallel rows (det <= 1e-14*uu*ww + tiny) take s = 0 (kernels.py:99-100)
  const bool nonpar = det > add(mul(mul(1e-14, uu), ww), kTiny);
  const double s0 = nonpar ? clip_quot(sub(mul(uw, wr), mul(ur, ww)), det) : 0.0;
  const double tn = add(mul(uw, s0), wr);
  // t = tn/ww; t < 0 iff tn < 0; t > 1 iff tn/ww > 1 + 2^-53 (RN ties to the
  // even 1.0), decided exactly: for ww < tn < 2ww, tn - ww is exact
  // (Sterbenz) and ww*2^-53 is exact (ww > 1e-280).
  const bool neg = lt0(tn);
  const bool above = tn > ww && (tn >= mul(2.0, ww) || sub(tn, ww) > mul(ww, 0x1p-53));
  // second quotient: re-clamped s (t outside [0,1]) or t itself
  double n2 = tn, m2 = ww;
  if (neg) { n2 = -ur; m2 = uu; }
  if (above) { n2 = sub(uw, ur); m2 = uu; }
  const double q2 = clip_quot(n2, m2);
  const bool clamp_t = neg || above;
  const double s = clamp_t ? q2 : s0;
  const double t = clamp_t ? (above ? 1.0 : 0.0) : q2;
  return sqn((p1 + scale(u, s)) - (p2 + scale(w, t)));
}

// Minimum squared 15-feature distance of the staged pair (ccd.py:135-153).
// Each loop iteration carries two (point-triangle) or three (segment-segment)
// independent features so the scheduler can overlap their FP64 latencies.
#ifndef LTSG_ILP
#define LTSG_ILP 0
#endif

template <int kStride>
__device__ __forceinline__ double staged_dist_sq(const Staged<kStride>& st) {
  double best = __longlong_as_double(0x7ff0000000000000LL);
#if LTSG_ILP
#error "the ILP variant was retired"
#else
#pragma unroll 1
  for (int q = 0; q < 6; ++q) {
    const int pbase = q < 3 ? kStA + 3 * q : kStB + 3 * (q - 3);
    const int tbase = q < 3 ? kStB : kStA;
    const int ebase = q < 3 ? kStEB : kStEA;
    best = min_nonneg(best, pt_sq_staged(st, pbase, tbase, ebase));
  }
#pragma unroll 1
  for (int f = 0; f < 9; ++f) {
    const int i = f / 3, j = f - 3 * (f / 3);
    best = min_nonneg(best, ss_sq_uniform(st.v3(kStA + 3 * i), st.v3(kStEA + 3 * i), st.at(kStAA + i),
                                          st.v3(kStB + 3 * j), st.v3(kStEB + 3 * j), st.at(kStBB + j)));
  }
#endif
  return best;
}

// ---------------------------------------------------------------- lite stage
// A leaner stage for register/shared-memory-bound kernels: corners and
// squared edge lengths only (24 doubles per thread); edge vectors are
// recomputed from the corners where used -- the same subtraction, so the
// same bits.  Layout: A corners 0..8, B corners 9..17, |eA|^2 18..20,
// |eB|^2 21..23.
constexpr int kLiteA = 0, kLiteB = 9, kLiteAA = 18, kLiteBB = 21;
constexpr int kStagedLite = 24;

template <int kStride>
__device__ __forceinline__ void stage_pair_lite(const Staged<kStride>& st, const Tri& a, const Tri& b) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    st.put(kLiteA + 3 * k, a.v[k]);
    st.put(kLiteB + 3 * k, b.v[k]);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const V3 ea = a.v[(k + 1) % 3] - a.v[k];
    const V3 eb = b.v[(k + 1) % 3] - b.v[k];
    st.at(kLiteAA + k) = dot_simd(ea, ea);
    st.at(kLiteBB + k) = dot_simd(eb, eb);
  }
}

template <int kStride>
__device__ __forceinline__ V3 lite_edge(const Staged<kStride>& st, int base, int k) {
  const int k1 = k == 2 ? 0 : k + 1;
  return st.v3(base + 3 * k1) - st.v3(base + 3 * k);
}

template <int kStride>
__device__ __forceinline__ double pt_sq_lite(const Staged<kStride>& st, int pk, int tb) {
  const V3 p = st.v3(pk);
  const V3 a = st.v3(tb), b = st.v3(tb + 3), c = st.v3(tb + 6);
  const V3 ab = b - a;
  const V3 ac = neg(a - c);  // -(e2), e2 = v0 - v2
  const V3 ap = p - a, bp = p - b, cp = p - c;
  const double d1 = dot_simd(ab, ap), d2 = dot_simd(ac, ap);
  const double d3 = dot_simd(ab, bp), d4 = dot_simd(ac, bp);
  const double d5 = dot_simd(ab, cp), d6 = dot_simd(ac, cp);
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  const double vb = sub(mul(d5, d2), mul(d1, d6));
  const double va = sub(mul(d3, d6), mul(d5, d4));
  const double e43 = sub(d4, d3), e56 = sub(d5, d6);
  const bool in_a = le0(d1) && le0(d2);
  const bool in_b = ge0(d3) && d4 <= d3;
  const bool in_c = ge0(d6) && d5 <= d6;
  const bool on_ab = le0(vc) && ge0(d1) && le0(d3);
  const bool on_ac = le0(vb) && ge0(d2) && le0(d6);
  const bool on_bc = le0(va) && ge0(e43) && ge0(e56);
  const bool vertex = in_a || in_b || in_c;
  const double den = add(add(va, vb), vc);
  int pv = 0, de = 0;
  double n1 = vb, m1 = den;
  bool face = true;
  if (on_bc) { n1 = e43; m1 = add(e43, e56); pv = 1; de = 1; face = false; }
  if (on_ac) { n1 = d2; m1 = sub(d2, d6); pv = 0; de = 2; face = false; }
  if (on_ab) { n1 = d1; m1 = sub(d1, d3); pv = 0; de = 0; face = false; }
  if (vertex) { pv = in_a ? 0 : (in_b ? 1 : 2); face = false; }
  double s1 = 0.0, s2 = 0.0;
  if (!vertex) s1 = sdiv(n1, m1);
  if (face) s2 = sdiv(vc, den);
  const V3 P = st.v3(tb + 3 * pv);
  V3 D1 = lite_edge(st, tb, de);
  if (de == 2) D1 = neg(D1);
  const V3 q = (P + scale(D1, s1)) + scale(ac, s2);
  return sqn(p - q);
}

template <int kStride>
__device__ __forceinline__ double staged_dist_sq_lite(const Staged<kStride>& st) {
  double best = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll 1
  for (int q = 0; q < 6; ++q) {
    const int pbase = q < 3 ? kLiteA + 3 * q : kLiteB + 3 * (q - 3);
    const int tbase = q < 3 ? kLiteB : kLiteA;
    best = min_nonneg(best, pt_sq_lite(st, pbase, tbase));
  }
#pragma unroll 1
  for (int i = 0; i < 3; ++i) {
    const V3 p1 = st.v3(kLiteA + 3 * i);
    const V3 u = lite_edge(st, kLiteA, i);
    const double uu = st.at(kLiteAA + i);
#pragma unroll 1
    for (int j = 0; j < 3; ++j)
      best = min_nonneg(best, ss_sq_uniform(p1, u, uu, st.v3(kLiteB + 3 * j), lite_edge(st, kLiteB, j),
                                            st.at(kLiteBB + j)));
  }
  return best;
}

}  // namespace ltsg
