// Exact-rounding FP64 geometry for the narrow phase (sm_100a).
//
// Every function reproduces, operation for operation, what the reference
// (ltsdem, numpy) evaluates, so results are bit-identical to it:
//   * plain products/sums never contract to FMA (explicit __dmul_rn/__dadd_rn;
//     the library is also compiled with -fmad=false);
//   * einsum row dots on C-contiguous rows sum (x0*y0 + x2*y2) + x1*y1
//     (dot_simd); on the broadcast operands of ccd._closest_feature they sum
//     sequentially (dot_seq);
//   * OpenBLAS ddot/dgemm are FMA chains fma(x2,y2, fma(x1,y1, x0*y0))
//     (dot_blas); the 3x3 dgemv is fma(m2,v2, fma(m0,v0, m1*v1)) (dot_gemv);
//   * np.linalg.norm(axis=1) is sqrt((x0^2 + x1^2) + x2^2).
// See oracle/fpexact.py for how these orders were established and pinned.
//
// Reference sources restated here (paths under /root/reference/pkg/src/ltsdem):
//   point_triangle_closest   kernels.py:23-75
//   segment_segment_closest  kernels.py:78-115
//   _feature_distances       ccd.py:135-153
//   _closest_feature         ccd.py:156-174
//   _face_normal             ccd.py:177-180
//   triangle_overlap_centroid kernels.py:138-201
//   _Motion.rotations / triangles_at  ccd.py:116-132
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ltsg {

#define LTSG_HD __host__ __device__ __forceinline__

constexpr double kTiny = 1e-300;      // kernels.py:12
constexpr double kWiden = 1e-3;       // ccd.py:29
constexpr double kRestSlop = 1e-9;    // ccd.py:30
constexpr int kMinSamples = 2;        // ccd.py:31
constexpr int kMaxSamples = 33;       // ccd.py:32
constexpr int kZoomSamples = 17;      // ccd.py:33
constexpr double kGrazeTol = 1e-9;    // ccd.py:34
constexpr int kBisectIters = 52;      // ccd.py:35
constexpr double kParallelCos = 1.0 - 1e-3;  // ccd.py:36

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ V3 v3(double x, double y, double z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return V3{sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return V3{add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
__device__ __forceinline__ V3 neg(V3 a) { return V3{-a.x, -a.y, -a.z}; }
__device__ __forceinline__ V3 scale(V3 a, double s) { return V3{mul(a.x, s), mul(a.y, s), mul(a.z, s)}; }

// einsum 'ij,ij->i' on C-contiguous rows
__device__ __forceinline__ double dot_simd(V3 u, V3 v) {
  return add(add(mul(u.x, v.x), mul(u.z, v.z)), mul(u.y, v.y));
}
// einsum on non-contiguous rows
__device__ __forceinline__ double dot_seq(V3 u, V3 v) {
  return add(add(mul(u.x, v.x), mul(u.y, v.y)), mul(u.z, v.z));
}
// OpenBLAS ddot, n = 3
__device__ __forceinline__ double dot_blas(V3 u, V3 v) {
  return fma_(u.z, v.z, fma_(u.y, v.y, mul(u.x, v.x)));
}
// OpenBLAS dgemv row (3x3 @ 3)
__device__ __forceinline__ double dot_gemv(V3 m, V3 v) {
  return fma_(m.z, v.z, fma_(m.x, v.x, mul(m.y, v.y)));
}
// squared np.linalg.norm(axis=1)
__device__ __forceinline__ double sqn(V3 w) {
  return add(add(mul(w.x, w.x), mul(w.y, w.y)), mul(w.z, w.z));
}
__device__ __forceinline__ double norm_blas(V3 w) { return __dsqrt_rn(dot_blas(w, w)); }
// np.cross
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return V3{sub(mul(a.y, b.z), mul(a.z, b.y)), sub(mul(a.z, b.x), mul(a.x, b.z)),
            sub(mul(a.x, b.y), mul(a.y, b.x))};
}

__device__ __forceinline__ double sdiv(double num, double den) {  // kernels._safe_div
  return dv(num, fabs(den) > kTiny ? den : 1.0);
}
__device__ __forceinline__ double clip01(double x) {  // np.clip(x, 0, 1), nan-propagating
  if (x != x) return x;
  double y = x > 0.0 ? x : 0.0;
  return y < 1.0 ? y : 1.0;
}

// Region codes of the Voronoi classification (priority: vertex a > b > c >
// edge ab > ac > bc > face), kernels.py:49-72.
enum Region : int { kFace = 0, kEdgeBC = 1, kEdgeAC = 2, kEdgeAB = 3, kVertC = 4, kVertB = 5, kVertA = 6 };

// Closest point on triangle (a,b,c) to p.  ab = b-a, ac = c-a, bc = c-b are
// passed in because they are per-triangle (and equal to what numpy computes
// per row).  Returns |p - closest|^2 in the reference's summation order.
template <bool kSeqDot, bool kWantPoint>
__device__ __forceinline__ double point_triangle_sq(V3 p, V3 a, V3 b, V3 c, V3 ab, V3 ac, V3 bc,
                                                    V3* closest = nullptr, int* region = nullptr) {
  auto dot = [](V3 u, V3 v) { return kSeqDot ? dot_seq(u, v) : dot_simd(u, v); };
  const V3 ap = p - a;
  const double d1 = dot(ab, ap);
  const double d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    if (kWantPoint) { *closest = a; *region = kVertA; }
    return sqn(ap);
  }
  const V3 bp = p - b;
  const double d3 = dot(ab, bp);
  const double d4 = dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) {
    if (kWantPoint) { *closest = b; *region = kVertB; }
    return sqn(bp);
  }
  const V3 cp = p - c;
  const double d5 = dot(ab, cp);
  const double d6 = dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) {
    if (kWantPoint) { *closest = c; *region = kVertC; }
    return sqn(cp);
  }
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  V3 q;
  int reg;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    const double w = sdiv(d1, sub(d1, d3));
    q = a + scale(ab, w);
    reg = kEdgeAB;
  } else {
    const double vb = sub(mul(d5, d2), mul(d1, d6));
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
      const double w = sdiv(d2, sub(d2, d6));
      q = a + scale(ac, w);
      reg = kEdgeAC;
    } else {
      const double va = sub(mul(d3, d6), mul(d5, d4));
      const double e43 = sub(d4, d3);
      const double e56 = sub(d5, d6);
      if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {
        const double w = sdiv(e43, add(e43, e56));
        q = b + scale(bc, w);
        reg = kEdgeBC;
      } else {
        const double den = add(add(va, vb), vc);
        const double v = sdiv(vb, den);
        const double w = sdiv(vc, den);
        q = (a + scale(ab, v)) + scale(ac, w);
        reg = kFace;
      }
    }
  }
  if (kWantPoint) { *closest = q; *region = reg; }
  return sqn(p - q);
}

// Clamped closest points of segments [p1, p1+u] and [p2, p2+w]; uu = |u|^2,
// ww = |w|^2 in dot_simd order.  Returns |c1 - c2|^2.
template <bool kWantPoints>
__device__ __forceinline__ double segment_segment_sq(V3 p1, V3 u, double uu, V3 p2, V3 w, double ww,
                                                     V3* c1 = nullptr, V3* c2 = nullptr) {
  const V3 r = p1 - p2;
  const double wr = dot_simd(w, r);
  const double ur = dot_simd(u, r);
  const double uw = dot_simd(u, w);
  const double det = sub(mul(uu, ww), mul(uw, uw));
  double s = clip01(sdiv(sub(mul(uw, wr), mul(ur, ww)), det));
  if (!(det > add(mul(mul(1e-14, uu), ww), kTiny))) s = 0.0;
  double t = sdiv(add(mul(uw, s), wr), ww);
  if (t < 0.0) {
    s = clip01(sdiv(-ur, uu));
  } else if (t > 1.0) {
    s = clip01(sdiv(sub(uw, ur), uu));
  }
  t = clip01(t);
  const bool u_dead = uu <= kTiny;
  const bool w_dead = ww <= kTiny;
  if (u_dead) {
    s = 0.0;
    t = clip01(sdiv(wr, ww));
  }
  if (w_dead) t = 0.0;
  if (w_dead && !u_dead) s = clip01(sdiv(-ur, uu));
  const V3 q1 = p1 + scale(u, s);
  const V3 q2 = p2 + scale(w, t);
  if (kWantPoints) { *c1 = q1; *c2 = q2; }
  return sqn(q1 - q2);
}

struct Tri {
  V3 v[3];
};

// Per-triangle quantities shared by all features: edges e_k = v[k+1] - v[k]
// (ccd._EDGE_A/_NEXT) and their squared lengths in dot_simd order.
struct TriPre {
  V3 v[3];
  V3 e[3];
  double ee[3];
};

__device__ __forceinline__ TriPre prep(const Tri& t) {
  TriPre p;
#pragma unroll
  for (int k = 0; k < 3; ++k) p.v[k] = t.v[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    p.e[k] = t.v[(k + 1) % 3] - t.v[k];
    p.ee[k] = dot_simd(p.e[k], p.e[k]);
  }
  return p;
}

// ccd._feature_distances for one row, squared: min over the six
// vertex-triangle and nine edge-edge features.  ab = e0, ac = -e2 = v2-v0
// (exact negation), bc = e1.
__device__ __forceinline__ double feature_dist_sq(const TriPre& A, const TriPre& B) {
  double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  {
    const V3 ab = B.e[0], ac = neg(B.e[2]), bc = B.e[1];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      best = fmin(best, point_triangle_sq<false, false>(A.v[k], B.v[0], B.v[1], B.v[2], ab, ac, bc));
  }
  {
    const V3 ab = A.e[0], ac = neg(A.e[2]), bc = A.e[1];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      best = fmin(best, point_triangle_sq<false, false>(B.v[k], A.v[0], A.v[1], A.v[2], ab, ac, bc));
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
      best = fmin(best, segment_segment_sq<false>(A.v[i], A.e[i], A.ee[i], B.v[j], B.e[j], B.ee[j]));
  }
  return best;
}

// sqrt is monotone and correctly rounded, so sqrt(min d^2) == min sqrt(d^2):
// the row distance is bit-identical to the reference's min over norms.
__device__ __forceinline__ double feature_dist(const Tri& a, const Tri& b) {
  return __dsqrt_rn(feature_dist_sq(prep(a), prep(b)));
}

// ccd._closest_feature: distance and witness points of the argmin feature.
// Point-triangle dots are sequential (broadcast operands), argmin picks the
// first minimal feature, vertex-triangle wins ties (ccd.py:170).
__device__ inline double closest_feature(const Tri& ta, const Tri& tb, V3* pa, V3* pb) {
  const TriPre A = prep(ta), B = prep(tb);
  double best_vt = 0.0;
  int arg_vt = -1;
  V3 cvt{0, 0, 0};
  for (int q = 0; q < 6; ++q) {
    const TriPre& P = q < 3 ? A : B;
    const TriPre& T = q < 3 ? B : A;
    const V3 p = P.v[q % 3];
    V3 c;
    int reg;
    const double d = __dsqrt_rn(point_triangle_sq<true, true>(
        p, T.v[0], T.v[1], T.v[2], T.e[0], neg(T.e[2]), T.e[1], &c, &reg));
    if (arg_vt < 0 || d < best_vt) {
      best_vt = d;
      arg_vt = q;
      cvt = c;
    }
  }
  double best_ee = 0.0;
  int arg_ee = -1;
  V3 e1{0, 0, 0}, e2{0, 0, 0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      V3 c1, c2;
      const double d = __dsqrt_rn(segment_segment_sq<true>(A.v[i], A.e[i], A.ee[i], B.v[j], B.e[j],
                                                           B.ee[j], &c1, &c2));
      if (arg_ee < 0 || d < best_ee) {
        best_ee = d;
        arg_ee = 3 * i + j;
        e1 = c1;
        e2 = c2;
      }
    }
  if (best_vt <= best_ee) {
    if (arg_vt < 3) {
      *pa = A.v[arg_vt];
      *pb = cvt;
    } else {
      *pa = cvt;
      *pb = B.v[arg_vt - 3];
    }
    return best_vt;
  }
  *pa = e1;
  *pb = e2;
  return best_ee;
}

__device__ __forceinline__ V3 face_normal(const Tri& t) {  // ccd._face_normal
  const V3 n = cross(t.v[1] - t.v[0], t.v[2] - t.v[0]);
  const double len = norm_blas(n);
  if (len > 0.0) return V3{dv(n.x, len), dv(n.y, len), dv(n.z, len)};
  return V3{0.0, 0.0, 1.0};
}

__device__ __forceinline__ V3 mean3(const Tri& t) {  // (3,3).mean(axis=0)
  return V3{dv(add(add(t.v[0].x, t.v[1].x), t.v[2].x), 3.0),
            dv(add(add(t.v[0].y, t.v[1].y), t.v[2].y), 3.0),
            dv(add(add(t.v[0].z, t.v[1].z), t.v[2].z), 3.0)};
}

// numpy 1-D float64 sum (pairwise_sum: sequential below 8 terms, else 8 lanes)
__device__ inline double np_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = add(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = add(r[j], a[i + j]);
  double res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
  for (; i < n; ++i) res = add(res, a[i]);
  return res;
}

constexpr int kMaxPoly = 48;

// kernels.triangle_overlap_centroid; returns false for None.
__device__ inline bool overlap_centroid(const Tri& ta, const Tri& tb, V3 normal, V3* out) {
  const double ln = norm_blas(normal);
  const V3 n{dv(normal.x, ln), dv(normal.y, ln), dv(normal.z, ln)};
  const V3 helper = fabs(n.x) < 0.9 ? V3{1.0, 0.0, 0.0} : V3{0.0, 1.0, 0.0};
  V3 u = cross(n, helper);
  const double lu = norm_blas(u);
  u = V3{dv(u.x, lu), dv(u.y, lu), dv(u.z, lu)};
  const V3 v = cross(n, u);
  const V3 origin = mean3(ta);

  double px[2][kMaxPoly], py[2][kMaxPoly];
  int np_ = 3;
  double cx[3], cy[3];
  for (int k = 0; k < 3; ++k) {
    const V3 rb = tb.v[k] - origin;
    px[0][k] = dot_blas(rb, u);
    py[0][k] = dot_blas(rb, v);
    const V3 ra = ta.v[k] - origin;
    cx[k] = dot_blas(ra, u);
    cy[k] = dot_blas(ra, v);
  }
  {
    const double e1x = sub(cx[1], cx[0]), e1y = sub(cy[1], cy[0]);
    const double e2x = sub(cx[2], cx[0]), e2y = sub(cy[2], cy[0]);
    if (sub(mul(e1x, e2y), mul(e1y, e2x)) < 0.0) {
      double t = cx[0]; cx[0] = cx[2]; cx[2] = t;
      t = cy[0]; cy[0] = cy[2]; cy[2] = t;
    }
  }
  int cur = 0;
  for (int i = 0; i < 3; ++i) {
    if (np_ == 0) return false;
    const double bx = cx[i], by = cy[i];
    const double ex = sub(cx[(i + 1) % 3], bx), ey = sub(cy[(i + 1) % 3], by);
    int nn = 0;
    const int nxt = cur ^ 1;
    for (int j = 0; j < np_; ++j) {
      const int jp = j == 0 ? np_ - 1 : j - 1;
      const double qx = px[cur][j], qy = py[cur][j];
      const double rx = px[cur][jp], ry = py[cur][jp];
      const bool cin = sub(mul(ex, sub(qy, by)), mul(ey, sub(qx, bx))) >= -1e-12;
      const bool pin = sub(mul(ex, sub(ry, by)), mul(ey, sub(rx, bx))) >= -1e-12;
      if (cin != pin) {
        const double dx = sub(qx, rx), dy = sub(qy, ry);
        const double den = sub(mul(ex, dy), mul(ey, dx));
        if (fabs(den) > kTiny) {
          const double lam = dv(sub(mul(ex, sub(by, ry)), mul(ey, sub(bx, rx))), -den);
          const double lc = clip01(lam);
          if (nn < kMaxPoly) {
            px[nxt][nn] = add(rx, mul(lc, dx));
            py[nxt][nn] = add(ry, mul(lc, dy));
          }
          ++nn;
        }
      }
      if (cin) {
        if (nn < kMaxPoly) {
          px[nxt][nn] = qx;
          py[nxt][nn] = qy;
        }
        ++nn;
      }
    }
    np_ = nn < kMaxPoly ? nn : kMaxPoly;
    cur = nxt;
  }
  if (np_ < 3) return false;
  double crs[kMaxPoly], tx[kMaxPoly], ty[kMaxPoly];
  for (int k = 0; k < np_; ++k) {
    const int kn = k + 1 == np_ ? 0 : k + 1;
    const double x = px[cur][k], y = py[cur][k], xn = px[cur][kn], yn = py[cur][kn];
    crs[k] = sub(mul(x, yn), mul(xn, y));
  }
  const double area = mul(0.5, np_sum(crs, np_));
  double c0, c1;
  if (fabs(area) < 1e-18) {
    double sx = px[cur][0], sy = py[cur][0];
    for (int k = 1; k < np_; ++k) {
      sx = add(sx, px[cur][k]);
      sy = add(sy, py[cur][k]);
    }
    c0 = dv(sx, (double)np_);
    c1 = dv(sy, (double)np_);
  } else {
    for (int k = 0; k < np_; ++k) {
      const int kn = k + 1 == np_ ? 0 : k + 1;
      tx[k] = mul(add(px[cur][k], px[cur][kn]), crs[k]);
      ty[k] = mul(add(py[cur][k], py[cur][kn]), crs[k]);
    }
    const double six_area = mul(6.0, area);
    c0 = dv(np_sum(tx, np_), six_area);
    c1 = dv(np_sum(ty, np_), six_area);
  }
  double la[3], lb[3];
  for (int k = 0; k < 3; ++k) {
    la[k] = dot_gemv(ta.v[k] - origin, n);
    lb[k] = dot_gemv(tb.v[k] - origin, n);
  }
  const double mid = add(mul(0.5, dv(add(add(la[0], la[1]), la[2]), 3.0)),
                         mul(0.5, dv(add(add(lb[0], lb[1]), lb[2]), 3.0)));
  *out = ((origin + scale(u, c0)) + scale(v, c1)) + scale(n, mid);
  return true;
}

// ---------------------------------------------------------------- motion

// Per-body free-flight constants, computed on the device from the raw
// snapshot exactly as ccd._Motion does (ccd.py:87-96, quaternions.py:54-63).
struct Motion {
  double x0[3];
  double v[3];
  double omega;      // |angular velocity| via ddot
  double K[9];       // cross-product matrix of the unit axis (row-major)
  double KK[9];      // K @ K (dgemm FMA chain)
  double base[9];    // to_matrix(q)
  int spinning;      // omega > 0
  int pad;
};

// Rotation at tau and world corners of a body-frame triangle (ccd.py:116-132).
__device__ __forceinline__ void rotation_at(const Motion& m, double tau, double R[9]) {
  if (!m.spinning) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = m.base[k];
    return;
  }
  const double ang = mul(m.omega, tau);
  double s, co;
  sincos(ang, &s, &co);
  const double c = sub(1.0, co);
  double M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = add(add(i == j ? 1.0 : 0.0, mul(s, m.K[3 * i + j])), mul(c, m.KK[3 * i + j]));
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      R[3 * i + j] = fma_(M[3 * i + 2], m.base[6 + j], fma_(M[3 * i + 1], m.base[3 + j], mul(M[3 * i], m.base[j])));
}

__device__ __forceinline__ Tri world_tri(const double R[9], const double pos[3], const double L[9]) {
  Tri t;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const double lx = L[3 * p], ly = L[3 * p + 1], lz = L[3 * p + 2];
    t.v[p].x = add(add(add(mul(R[0], lx), mul(R[2], lz)), mul(R[1], ly)), pos[0]);
    t.v[p].y = add(add(add(mul(R[3], lx), mul(R[5], lz)), mul(R[4], ly)), pos[1]);
    t.v[p].z = add(add(add(mul(R[6], lx), mul(R[8], lz)), mul(R[7], ly)), pos[2]);
  }
  return t;
}

__device__ __forceinline__ void position_at(const Motion& m, double tau, double pos[3]) {
  pos[0] = add(m.x0[0], mul(tau, m.v[0]));
  pos[1] = add(m.x0[1], mul(tau, m.v[1]));
  pos[2] = add(m.x0[2], mul(tau, m.v[2]));
}

// np.linspace(start, stop, n)[i] (numpy 2.x): step = (stop-start)/(n-1),
// g[i] = i*step + start, g[n-1] = stop; a zero step uses (i/(n-1))*delta.
__device__ __forceinline__ double linspace_at(double start, double stop, int n, int i) {
  if (n <= 1) return start;
  if (i == n - 1) return stop;
  const double div = (double)(n - 1);
  const double delta = sub(stop, start);
  const double step = dv(delta, div);
  if (step == 0.0) return add(mul(dv((double)i, div), delta), start);
  return add(mul((double)i, step), start);
}

}  // namespace ltsg
