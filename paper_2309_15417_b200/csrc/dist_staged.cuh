// The 15-feature triangle-pair distance over shared-memory-staged triangles.
//
// Same arithmetic as geom.cuh's feature_dist (bit-identical results), laid
// out for throughput on sm_100a:
//  * the two world triangles, their edge vectors and squared edge lengths are
//    staged once per row in shared memory, structure-of-arrays across the
//    block's threads (element k of thread t at s[k * stride + t], so a warp's
//    accesses are conflict-free), and computed once instead of once per
//    feature;
//  * the six point-triangle and nine segment-segment features run as two
//    compact loops (not unrolled): one copy of each feature's code keeps the
//    kernel inside the instruction cache;
//  * divisions are skipped wherever their rounded quotient cannot change the
//    result: a clamped parameter whose numerator lies outside (0, den) is
//    exactly 0 or 1 after the clamp, and t > 1 is decided exactly without
//    dividing (see seg_param below).  Both choices are proven per case in
//    the comments and checked bit-for-bit against the reference's rows.
#pragma once

#include "geom.cuh"

namespace ltsg {

// Staged row layout (doubles): A corners 0..8, B corners 9..17, A edges
// 18..26, B edges 27..35, |eA|^2 36..38, |eB|^2 39..41.
constexpr int kStA = 0, kStB = 9, kStEA = 18, kStEB = 27, kStAA = 36, kStBB = 39;
constexpr int kStaged = 42;

struct Staged {
  double* s;
  int stride;
  __device__ __forceinline__ double& at(int k) const { return s[k * stride]; }
  __device__ __forceinline__ V3 v3(int k) const { return V3{at(k), at(k + 1), at(k + 2)}; }
  __device__ __forceinline__ void put(int k, V3 v) const {
    at(k) = v.x;
    at(k + 1) = v.y;
    at(k + 2) = v.z;
  }
};

// Stage triangles a, b: corners, edges e_k = v[k+1] - v[k] and |e_k|^2 in
// dot_simd order (the reference computes both per feature; same values).
__device__ __forceinline__ void stage_pair(const Staged& st, const Tri& a, const Tri& b) {
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

// clip01(num / den) for den > 0, as np.clip(_safe_div(num, den), 0, 1):
// num <= 0 gives a quotient <= 0 (or -0) which clips to +0; num >= den gives
// a quotient >= 1 which clips to 1; only 0 < num < den needs the division.
// Requires den > 1e-300 so that _safe_div divides by den itself.
__device__ __forceinline__ double clip_quot(double num, double den) {
  if (!(num > 0.0)) return num != num ? num : 0.0;
  if (num >= den) return 1.0;
  return dv(num, den);
}

// Squared distance of segments (kernels.py:78-115) with the division
// shortcuts.  u, w edge vectors; uu, ww their squared lengths.
__device__ __forceinline__ double seg_sq_fast(V3 p1, V3 u, double uu, V3 p2, V3 w, double ww) {
  const bool u_ok = uu > kTiny, w_ok = ww > kTiny;
  if (!u_ok || !w_ok) return segment_segment_sq<false>(p1, u, uu, p2, w, ww);
  const V3 r = p1 - p2;
  const double wr = dot_simd(w, r);
  const double ur = dot_simd(u, r);
  const double uw = dot_simd(u, w);
  const double det = sub(mul(uu, ww), mul(uw, uw));
  double s = 0.0;
  // det > thr > 0 there, so _safe_div divides by det
  if (det > add(mul(mul(1e-14, uu), ww), kTiny)) s = clip_quot(sub(mul(uw, wr), mul(ur, ww)), det);
  const double tn = add(mul(uw, s), wr);
  double t;
  if (tn < 0.0) {  // t < 0: re-clamp s from -ur/uu, t clips to 0
    s = clip_quot(-ur, uu);
    t = 0.0;
  } else {
    // t > 1 exactly when RN(tn/ww) > 1, i.e. tn/ww > 1 + 2^-53 (ties round to
    // the even 1.0).  For ww < tn < 2ww, tn - ww is exact (Sterbenz) and
    // ww * 2^-53 is exact, so the comparison is exact.
    bool above;
    if (!(tn > ww)) above = false;
    else if (tn >= mul(2.0, ww)) above = true;
    else above = sub(tn, ww) > mul(ww, 0x1p-53);
    if (above) {
      s = clip_quot(sub(uw, ur), uu);
      t = 1.0;
    } else {
      t = tn == 0.0 ? 0.0 : clip01(dv(tn, ww));
    }
  }
  const V3 q1 = p1 + scale(u, s);
  const V3 q2 = p2 + scale(w, t);
  return sqn(q1 - q2);
}

// Squared point-triangle distance (kernels.py:23-75), edges from the stage:
// ab = e0, ac = -e2 (exact negation of v0 - v2), bc = e1.
__device__ __forceinline__ double pt_sq_fast(V3 p, V3 a, V3 b, V3 c, V3 ab, V3 ac, V3 bc) {
  const V3 ap = p - a;
  const double d1 = dot_simd(ab, ap);
  const double d2 = dot_simd(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return sqn(ap);
  const V3 bp = p - b;
  const double d3 = dot_simd(ab, bp);
  const double d4 = dot_simd(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return sqn(bp);
  const V3 cp = p - c;
  const double d5 = dot_simd(ab, cp);
  const double d6 = dot_simd(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return sqn(cp);
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  V3 q;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    q = a + scale(ab, sdiv(d1, sub(d1, d3)));
  } else {
    const double vb = sub(mul(d5, d2), mul(d1, d6));
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
      q = a + scale(ac, sdiv(d2, sub(d2, d6)));
    } else {
      const double va = sub(mul(d3, d6), mul(d5, d4));
      const double e43 = sub(d4, d3);
      const double e56 = sub(d5, d6);
      if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {
        q = b + scale(bc, sdiv(e43, add(e43, e56)));
      } else {
        const double den = add(add(va, vb), vc);
        q = (a + scale(ab, sdiv(vb, den))) + scale(ac, sdiv(vc, den));
      }
    }
  }
  return sqn(p - q);
}

// Minimum squared 15-feature distance of the staged pair.
__device__ __forceinline__ double staged_dist_sq(const Staged& st) {
  double best = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll 1
  for (int q = 0; q < 6; ++q) {
    const int pbase = q < 3 ? kStA + 3 * q : kStB + 3 * (q - 3);
    const int tbase = q < 3 ? kStB : kStA;
    const int ebase = q < 3 ? kStEB : kStEA;
    const V3 p = st.v3(pbase);
    const V3 a = st.v3(tbase), b = st.v3(tbase + 3), c = st.v3(tbase + 6);
    const V3 ab = st.v3(ebase), bc = st.v3(ebase + 3), ac = neg(st.v3(ebase + 6));
    best = fmin(best, pt_sq_fast(p, a, b, c, ab, ac, bc));
  }
#pragma unroll 1
  for (int f = 0; f < 9; ++f) {
    const int i = f / 3, j = f - 3 * (f / 3);
    best = fmin(best, seg_sq_fast(st.v3(kStA + 3 * i), st.v3(kStEA + 3 * i), st.at(kStAA + i),
                                  st.v3(kStB + 3 * j), st.v3(kStEB + 3 * j), st.at(kStBB + j)));
  }
  return best;
}

}  // namespace ltsg
