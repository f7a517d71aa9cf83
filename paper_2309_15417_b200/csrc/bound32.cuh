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
