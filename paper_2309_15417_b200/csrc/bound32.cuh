// Certified FP32 upper bound on the reference's 15-feature distance
// (ccd._feature_distances, ccd.py:135-153), used to decide rows whose
// distance is certainly at or below a threshold without the bit-exact FP64
// evaluation.
//
// Why it is an upper bound.  The reference's distance is the minimum over
// its 15 features, so it is at most any one feature's value.  Its six
// point-triangle features evaluate, for a vertex p of one triangle, the
// Voronoi-region closest point of the other (kernels.py:23-75): for a
// non-sliver triangle that is the true closest point up to rounding, so the
// feature value is dist(p, T) up to a relative error far below 1e-7
// (conditioning <= 1e4 for non-slivers, FP64 rounding 1e-16).  And
// dist(p, T) <= |p - x| for every point x of T.  Here x is the closest
// point computed in FP32: the closest of the three clamped edge points
// (exactly points of the FP32 edges), or the plane projection when the FP32
// inside test passes.  The returned bound U satisfies
//     reference distance <= U + margin,
//     margin = (kBoundRel + fe) * s + kCullMargin * s_world,
// s the largest |coordinate - origin| of the pair in the local frame the FP32
// arithmetic runs in.  First-order rounding analysis (u = 2^-24):
//   * rounding the local FP64 coordinates to FP32 moves each triangle by at
//     most sqrt(3) u s;
//   * an edge candidate (clamped parameter, FMA residual, dot, sqrt) is
//     within ~10 u s of the distance to a true edge point;
//   * a face candidate divides by |n| = 2 area, whose FP32 value carries an
//     absolute error ~12 u s^2: its relative error, and the error of the
//     inside test (a projection misjudged inside lies within that error of
//     the triangle), are covered by fe = 64 u s^2 / |n| per triangle; a
//     triangle with fe > 1e-3 does not use its face candidate.
// kBoundRel = 2e-5 covers the ~16 u s of the first two items 20x; s_world
// (world coordinate scale) carries the reference's own FP64 rounding, as for
// the culls.  Rows within the margin of a threshold -- and every row
// involving a sliver (record radius -1) or extents outside [1e-9, 1e9] --
// are left to the exact evaluation.  Decisions taken from the bound are the
// reference's decisions; distances themselves are never taken from it.
#pragma once

namespace ltsg {

constexpr double kBoundRel = 2e-5;

struct F3 {
  float x, y, z;
};

__device__ __forceinline__ F3 f3sub(F3 a, F3 b) { return F3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ float f3dot(F3 a, F3 b) { return __fmaf_rn(a.z, b.z, __fmaf_rn(a.y, b.y, a.x * b.x)); }
__device__ __forceinline__ F3 f3cross(F3 a, F3 b) {
  return F3{__fmaf_rn(a.y, b.z, -a.z * b.y), __fmaf_rn(a.z, b.x, -a.x * b.z), __fmaf_rn(a.x, b.y, -a.y * b.x)};
}

struct TriF {
  F3 v[3];
  F3 e[3];     // e[k] = v[k+1] - v[k]
  float ie[3];  // 1 / |e[k]|^2 (0 for a zero-length edge)
  F3 n;        // e[0] x (v[2] - v[0])
  float inn;   // 1 / |n|^2 (0: no face candidate)
  float fe;    // relative error bound of the face candidate (see above)
};

// s: the pair's local coordinate scale
__device__ __forceinline__ TriF trif(F3 a, F3 b, F3 c, float s) {
  TriF t;
  t.v[0] = a;
  t.v[1] = b;
  t.v[2] = c;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    t.e[k] = f3sub(t.v[k == 2 ? 0 : k + 1], t.v[k]);
    const float ee = f3dot(t.e[k], t.e[k]);
    t.ie[k] = ee > 0.f ? __frcp_rn(ee) : 0.f;
  }
  t.n = f3cross(t.e[0], f3sub(c, a));
  const float nn = f3dot(t.n, t.n);
  t.inn = nn > 0.f ? __frcp_rn(nn) : 0.f;
  t.fe = nn > 0.f ? 64.f * 5.9604645e-8f * s * s * sqrtf(t.inn) : 1.f;
  if (!(t.fe <= 1e-3f)) {
    t.inn = 0.f;
    t.fe = 0.f;
  }
  return t;
}

// squared distance from p to (a point of) triangle t, in FP32
__device__ __forceinline__ float pt_ub_sq(F3 p, const TriF& t) {
  float best = 3.0e38f;
  bool inside = t.inn > 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const F3 w = f3sub(p, t.v[k]);
    const float s = fminf(fmaxf(f3dot(w, t.e[k]) * t.ie[k], 0.f), 1.f);
    const F3 r{__fmaf_rn(-s, t.e[k].x, w.x), __fmaf_rn(-s, t.e[k].y, w.y), __fmaf_rn(-s, t.e[k].z, w.z)};
    best = fminf(best, f3dot(r, r));
    inside = inside && f3dot(t.n, f3cross(t.e[k], w)) >= 0.f;
  }
  if (inside) {
    const float h = f3dot(f3sub(p, t.v[0]), t.n);
    best = fminf(best, h * h * t.inn);
  }
  return best;
}

// FP32 upper bound on the 15-feature distance of world triangles a, b (FP64
// corners), and its margin.  Returns false when the pair is outside the
// bound's domain (the caller evaluates exactly).
__device__ __forceinline__ bool feature_ub(const Tri& a, const Tri& b, double* ub, double* margin) {
  const double ox = a.v[0].x, oy = a.v[0].y, oz = a.v[0].z;
  float c[18];
  float sl = 0.f;
  double sw = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[3 * k] = (float)(a.v[k].x - ox);
    c[3 * k + 1] = (float)(a.v[k].y - oy);
    c[3 * k + 2] = (float)(a.v[k].z - oz);
    c[9 + 3 * k] = (float)(b.v[k].x - ox);
    c[9 + 3 * k + 1] = (float)(b.v[k].y - oy);
    c[9 + 3 * k + 2] = (float)(b.v[k].z - oz);
  }
#pragma unroll
  for (int k = 0; k < 18; ++k) sl = fmaxf(sl, fabsf(c[k]));
  sw = fabs(ox) + fabs(oy) + fabs(oz) + (double)sl;
  // FP32 range: extents within [1e-9, 1e9] keep every product (up to s^4) normal
  if (!(sl < 1e9f) || sl < 1e-9f) return false;
  // one side at a time keeps a single triangle's FP32 constants live
  float best = 3.0e38f, fe = 0.f;
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int t0 = side ? 0 : 9, p0 = side ? 9 : 0;
    const TriF t = trif(F3{c[t0], c[t0 + 1], c[t0 + 2]}, F3{c[t0 + 3], c[t0 + 4], c[t0 + 5]},
                        F3{c[t0 + 6], c[t0 + 7], c[t0 + 8]}, sl);
    fe = fmaxf(fe, t.fe);
#pragma unroll
    for (int k = 0; k < 3; ++k) best = fminf(best, pt_ub_sq(F3{c[p0 + 3 * k], c[p0 + 3 * k + 1], c[p0 + 3 * k + 2]}, t));
  }
  *ub = (double)sqrtf(best);
  *margin = (kBoundRel + (double)fe) * (double)sl + kCullMargin * sw;
  return true;
}

}  // namespace ltsg

// ---------------------------------------------------------------- FP32 guide
//
// The guide picks, in FP32, the feature most likely to be the row's minimum;
// the caller then evaluates THAT ONE feature with the reference's FP64
// arithmetic.  A row whose single exact feature is at or below its threshold
// is at or below it in the reference too (the reference takes the minimum
// over all 15, ccd.py:153), so the decision needs no error analysis: the
// guide can only cost time, never change a result.
namespace ltsg {

struct Guide {
  float d2;  // approximate squared distance of the picked feature
  int k;     // 0..2: corner k of a vs triangle b; 3..5: corner k-3 of b vs a;
             // 6 + 3 i + j: edge i of a vs edge j of b; -1: nothing usable
};

__device__ __forceinline__ float clamp01f(float x) { return fminf(fmaxf(x, 0.f), 1.f); }

// squared distance of segments [p1, p1 + u] and [p2, p2 + w] (clamped
// closest points, the construction of kernels.py:78-115, in FP32)
__device__ __forceinline__ float ss_guide_sq(F3 p1, F3 u, float uu, float iu, F3 p2, F3 w, float ww, float iw) {
  const F3 r = f3sub(p1, p2);
  const float wr = f3dot(w, r), ur = f3dot(u, r), uw = f3dot(u, w);
  const float det = __fmaf_rn(uu, ww, -uw * uw);
  float s = det > 1e-6f * uu * ww ? clamp01f(__fdividef(__fmaf_rn(uw, wr, -ur * ww), det)) : 0.f;
  float t = __fmaf_rn(uw, s, wr) * iw;
  s = t < 0.f ? clamp01f(-ur * iu) : (t > 1.f ? clamp01f((uw - ur) * iu) : s);
  t = clamp01f(t);
  const F3 d{__fmaf_rn(s, u.x, r.x) - t * w.x, __fmaf_rn(s, u.y, r.y) - t * w.y, __fmaf_rn(s, u.z, r.z) - t * w.z};
  return f3dot(d, d);
}

__device__ __forceinline__ float frcp(float x) { return __fdividef(1.f, x); }

// Per-triangle constants of the scalar guide: edges ab, ac, their Gram
// entries, the normal and reciprocals (0 for degenerate lengths).
struct GuideTri {
  F3 ab, ac, n;
  float AA, AC, CC, BB;      // ab.ab, ab.ac, ac.ac, |bc|^2
  float iAA, iCC, iBB, inn;  // reciprocals (0: unusable)
};

__device__ __forceinline__ GuideTri guide_tri(F3 a, F3 b, F3 c) {
  GuideTri t;
  t.ab = f3sub(b, a);
  t.ac = f3sub(c, a);
  t.n = f3cross(t.ab, t.ac);
  t.AA = f3dot(t.ab, t.ab);
  t.AC = f3dot(t.ab, t.ac);
  t.CC = f3dot(t.ac, t.ac);
  t.BB = fmaxf(t.AA - 2.f * t.AC + t.CC, 0.f);
  const float nn = f3dot(t.n, t.n);
  t.iAA = t.AA > 0.f ? frcp(t.AA) : 0.f;
  t.iCC = t.CC > 0.f ? frcp(t.CC) : 0.f;
  t.iBB = t.BB > 0.f ? frcp(t.BB) : 0.f;
  t.inn = nn > 1e-12f * t.AA * t.CC ? frcp(nn) : 0.f;
  return t;
}

// squared distance from p to the triangle, from scalars only: ap = p - a
// (P2 = |ap|^2).  Minimum over the three clamped edges, and the plane
// distance when all three barycentric numerators are non-negative.
__device__ __forceinline__ float pt_guide_sq(F3 ap, float P2, const GuideTri& t) {
  const float d1 = f3dot(t.ab, ap), d2 = f3dot(t.ac, ap);
  const float d3 = d1 - t.AA, d4 = d2 - t.AC, d5 = d1 - t.AC, d6 = d2 - t.CC;
  const float vc = __fmaf_rn(d1, d4, -d3 * d2), vb = __fmaf_rn(d5, d2, -d1 * d6), va = __fmaf_rn(d3, d6, -d5 * d4);
  const float tab = clamp01f(d1 * t.iAA), tac = clamp01f(d2 * t.iCC);
  const float e = d4 - d3, tbc = clamp01f(e * t.iBB);
  const float B2 = __fmaf_rn(-2.f, d1, P2) + t.AA;  // |p - b|^2
  float best = __fmaf_rn(tab, __fmaf_rn(tab, t.AA, -2.f * d1), P2);
  best = fminf(best, __fmaf_rn(tac, __fmaf_rn(tac, t.CC, -2.f * d2), P2));
  best = fminf(best, __fmaf_rn(tbc, __fmaf_rn(tbc, t.BB, -2.f * e), B2));
  const float h = f3dot(t.n, ap);
  if (va >= 0.f && vb >= 0.f && vc >= 0.f && t.inn > 0.f) best = fminf(best, h * h * t.inn);
  return fmaxf(best, 0.f);
}

// squared distance of segments [p1, p1 + u], [p2, p2 + w] from scalars:
// r = p1 - p2 (R2 = |r|^2), ur = u.r, wr = w.r, uw = u.w
__device__ __forceinline__ float ss_guide_scalar(float R2, float ur, float wr, float uw, float uu, float iu, float ww,
                                                 float iw) {
  const float det = __fmaf_rn(uu, ww, -uw * uw);
  float s = det > 1e-6f * uu * ww ? clamp01f(__fdividef(__fmaf_rn(uw, wr, -ur * ww), det)) : 0.f;
  float t = __fmaf_rn(uw, s, wr) * iw;
  s = t < 0.f ? clamp01f(-ur * iu) : (t > 1.f ? clamp01f((uw - ur) * iu) : s);
  t = clamp01f(t);
  // |r + s u - t w|^2
  const float d = R2 + s * __fmaf_rn(s, uu, 2.f * ur) + t * (__fmaf_rn(t, ww, -2.f * wr) - 2.f * s * uw);
  return fmaxf(d, 0.f);
}

// wa, wb: world records (9 corner doubles first).  kWithEdges adds the nine
// edge-edge features to the six corner-triangle ones.  Every feature value
// comes from the nine corner differences A_i - B_j, the edge vectors and
// per-triangle constants; cancellation in the expanded squares costs
// accuracy for distances far below the triangle size, which only makes the
// guess worse (see above: the guide decides nothing).
template <bool kWithEdges>
__device__ __forceinline__ Guide feature_guide(const double* wa, const double* wb) {
  const double ox = __ldg(wa), oy = __ldg(wa + 1), oz = __ldg(wa + 2);
  F3 A[3], B[3];
  float sl = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    A[k] = F3{(float)(__ldg(wa + 3 * k) - ox), (float)(__ldg(wa + 3 * k + 1) - oy), (float)(__ldg(wa + 3 * k + 2) - oz)};
    B[k] = F3{(float)(__ldg(wb + 3 * k) - ox), (float)(__ldg(wb + 3 * k + 1) - oy), (float)(__ldg(wb + 3 * k + 2) - oz)};
    sl = fmaxf(sl, fmaxf(fmaxf(fabsf(A[k].x), fabsf(A[k].y)), fabsf(A[k].z)));
    sl = fmaxf(sl, fmaxf(fmaxf(fabsf(B[k].x), fabsf(B[k].y)), fabsf(B[k].z)));
  }
  Guide g{3.0e38f, -1};
  if (!(sl < 1e9f) || sl < 1e-9f) return g;  // outside the FP32 range: no guess
  const GuideTri ta = guide_tri(A[0], A[1], A[2]);
  const GuideTri tb = guide_tri(B[0], B[1], B[2]);
  F3 D[3][3];
  float R2[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      D[i][j] = f3sub(A[i], B[j]);
      R2[i][j] = f3dot(D[i][j], D[i][j]);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // corner k of a against triangle b: ap = A_k - B_0
    const float d = pt_guide_sq(D[k][0], R2[k][0], tb);
    if (d < g.d2) g = Guide{d, k};
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // corner k of b against triangle a: ap = B_k - A_0
    const float d = pt_guide_sq(F3{-D[0][k].x, -D[0][k].y, -D[0][k].z}, R2[0][k], ta);
    if (d < g.d2) g = Guide{d, 3 + k};
  }
  if (kWithEdges) {
    // edges e_k = v[k+1] - v[k]: e0 = ab, e1 = ac - ab, e2 = -ac
    F3 ea[3] = {ta.ab, f3sub(ta.ac, ta.ab), F3{-ta.ac.x, -ta.ac.y, -ta.ac.z}};
    F3 eb[3] = {tb.ab, f3sub(tb.ac, tb.ab), F3{-tb.ac.x, -tb.ac.y, -tb.ac.z}};
    const float ua[3] = {ta.AA, ta.BB, ta.CC}, ia[3] = {ta.iAA, ta.iBB, ta.iCC};
    const float ub[3] = {tb.AA, tb.BB, tb.CC}, ib[3] = {tb.iAA, tb.iBB, tb.iCC};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float ur = f3dot(ea[i], D[i][j]), wr = f3dot(eb[j], D[i][j]), uw = f3dot(ea[i], eb[j]);
        const float d = ss_guide_scalar(R2[i][j], ur, wr, uw, ua[i], ia[i], ub[j], ib[j]);
        if (d < g.d2) g = Guide{d, 6 + 3 * i + j};
      }
    }
  }
  return g;
}

// Closest-point direction of feature k (numbered as in Guide) in FP32: the
// vector between the feature's approximate closest points.  Used only as a
// separating direction, so its accuracy affects the strength of the bound
// below, never its validity.
__device__ __forceinline__ F3 guide_direction(const double* wa, const double* wb, int k) {
  if (k < 6) {
    const double* pp = k < 3 ? wa + 3 * k : wb + 3 * (k - 3);
    const double* tt = k < 3 ? wb : wa;
    const double px = __ldg(pp), py = __ldg(pp + 1), pz = __ldg(pp + 2);
    F3 v[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      v[c] = F3{(float)(__ldg(tt + 3 * c) - px), (float)(__ldg(tt + 3 * c + 1) - py), (float)(__ldg(tt + 3 * c + 2) - pz)};
    // the query point is the origin: closest of the three clamped edge
    // points, or the plane projection when it falls inside
    float best = 3.0e38f;
    F3 dir{0.f, 0.f, 0.f};
    const F3 n = f3cross(f3sub(v[1], v[0]), f3sub(v[2], v[0]));
    bool inside = f3dot(n, n) > 0.f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const F3 e = f3sub(v[c == 2 ? 0 : c + 1], v[c]);
      const float ee = f3dot(e, e);
      const float s = ee > 0.f ? clamp01f(-f3dot(v[c], e) / ee) : 0.f;
      const F3 x{__fmaf_rn(s, e.x, v[c].x), __fmaf_rn(s, e.y, v[c].y), __fmaf_rn(s, e.z, v[c].z)};
      const float d = f3dot(x, x);
      if (d < best) {
        best = d;
        dir = x;
      }
      inside = inside && f3dot(n, f3cross(e, F3{-v[c].x, -v[c].y, -v[c].z})) >= 0.f;
    }
    if (inside) dir = n;  // the plane normal is the direction of the projection
    return dir;
  }
  const int i = (k - 6) / 3, j = (k - 6) % 3;
  const double* p1 = wa + 3 * i;
  const double* q1 = wa + 3 * (i == 2 ? 0 : i + 1);
  const double* p2 = wb + 3 * j;
  const double* q2 = wb + 3 * (j == 2 ? 0 : j + 1);
  const double ox = __ldg(p1), oy = __ldg(p1 + 1), oz = __ldg(p1 + 2);
  const F3 u{(float)(__ldg(q1) - ox), (float)(__ldg(q1 + 1) - oy), (float)(__ldg(q1 + 2) - oz)};
  const F3 b0{(float)(__ldg(p2) - ox), (float)(__ldg(p2 + 1) - oy), (float)(__ldg(p2 + 2) - oz)};
  const F3 b1{(float)(__ldg(q2) - ox), (float)(__ldg(q2 + 1) - oy), (float)(__ldg(q2 + 2) - oz)};
  const F3 w = f3sub(b1, b0);
  const F3 r{-b0.x, -b0.y, -b0.z};  // p1 - p2 with p1 at the origin
  const float uu = f3dot(u, u), ww = f3dot(w, w);
  const float iu = uu > 0.f ? 1.f / uu : 0.f, iw = ww > 0.f ? 1.f / ww : 0.f;
  const float wr = f3dot(w, r), ur = f3dot(u, r), uw = f3dot(u, w);
  const float det = __fmaf_rn(uu, ww, -uw * uw);
  float s = det > 1e-6f * uu * ww ? clamp01f(__fdividef(__fmaf_rn(uw, wr, -ur * ww), det)) : 0.f;
  float t = __fmaf_rn(uw, s, wr) * iw;
  s = t < 0.f ? clamp01f(-ur * iu) : (t > 1.f ? clamp01f((uw - ur) * iu) : s);
  t = clamp01f(t);
  return F3{__fmaf_rn(s, u.x, r.x) - t * w.x, __fmaf_rn(s, u.y, r.y) - t * w.y, __fmaf_rn(s, u.z, r.z) - t * w.z};
}

// Certified "above the threshold" from one separating direction.  For ANY
// direction u, the gap between the projections of the two triangles onto u,
// divided by |u|, is a lower bound of their distance -- the argument of
// sat_cull (search.cu), whose margin and sliver rule are used unchanged.
// The direction is the guide's closest-point direction, which makes the
// bound nearly tight when the guide found the closest features; a poor
// direction only makes the test fail.  FP64 projections on world corners.
__device__ __forceinline__ bool direction_cull(const double* wa, const double* wb, F3 dir, double thr) {
  const double ra = __ldg(wa + 15), rb = __ldg(wb + 15);
  if (ra < 0.0 || rb < 0.0) return false;  // slivers are never culled
  const double u0 = (double)dir.x, u1 = (double)dir.y, u2 = (double)dir.z;
  const double len = sqrt(fma(u0, u0, fma(u1, u1, u2 * u2)));
  if (!(len > 0.0) || !(len < 1e300)) return false;
  double scale = 1.0 + ra + rb;
#pragma unroll
  for (int k = 0; k < 3; ++k) scale += fabs(__ldg(wa + 12 + k)) + fabs(__ldg(wb + 12 + k));
  const double T = thr + kCullMargin * scale;
  double alo = 0.0, ahi = 0.0, blo = 0.0, bhi = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = fma(u0, __ldg(wa + 3 * k), fma(u1, __ldg(wa + 3 * k + 1), u2 * __ldg(wa + 3 * k + 2)));
    const double y = fma(u0, __ldg(wb + 3 * k), fma(u1, __ldg(wb + 3 * k + 1), u2 * __ldg(wb + 3 * k + 2)));
    alo = k ? fmin(alo, x) : x;
    ahi = k ? fmax(ahi, x) : x;
    blo = k ? fmin(blo, y) : y;
    bhi = k ? fmax(bhi, y) : y;
  }
  return fmax(blo - ahi, alo - bhi) > T * len;
}

}  // namespace ltsg
