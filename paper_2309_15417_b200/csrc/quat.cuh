// Unit-quaternion helpers with the reference's rounding (ltsdem.quaternions,
// quaternions.py): elementwise numpy arithmetic separately rounded, the
// 4-vector norm an OpenBLAS ddot FMA chain.  Shared by the broad phase
// (broad.cu) and the contact consumers (contacts.cu).
#pragma once

#include "geom.cuh"

namespace ltsg {

__device__ __forceinline__ double dot4_blas(const double a[4], const double b[4]) {
  return fma_(a[3], b[3], fma_(a[2], b[2], fma_(a[1], b[1], mul(a[0], b[0]))));
}

__device__ __forceinline__ void normalize4(double q[4]) {  // quaternions.normalize (:17-21)
  const double n = __dsqrt_rn(dot4_blas(q, q));
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = dv(q[k], n);
}

// quaternions.multiply (:24-35), left to right as written
__device__ __forceinline__ void qmul(const double p[4], const double q[4], double out[4]) {
  const double w1 = p[0], x1 = p[1], y1 = p[2], z1 = p[3];
  const double w2 = q[0], x2 = q[1], y2 = q[2], z2 = q[3];
  out[0] = sub(sub(sub(mul(w1, w2), mul(x1, x2)), mul(y1, y2)), mul(z1, z2));
  out[1] = sub(add(add(mul(w1, x2), mul(x1, w2)), mul(y1, z2)), mul(z1, y2));
  out[2] = add(add(sub(mul(w1, y2), mul(x1, z2)), mul(y1, w2)), mul(z1, x2));
  out[3] = add(sub(add(mul(w1, z2), mul(x1, y2)), mul(y1, x2)), mul(z1, w2));
}

// quaternions.advance (:85-90): normalize(multiply(from_rotation_vector(omega dt), q))
__device__ __forceinline__ void advance(const double q[4], V3 omega, double dt, double out[4]) {
  const V3 phi = scale(omega, dt);
  const double angle = norm_blas(phi);
  double dq[4];
  if (angle < 1e-12) {  // from_rotation_vector's series branch (:79-81)
    dq[0] = 1.0;
    dq[1] = mul(0.5, phi.x);
    dq[2] = mul(0.5, phi.y);
    dq[3] = mul(0.5, phi.z);
    normalize4(dq);
  } else {  // from_axis_angle (:66-72) with n = |phi| = angle
    const double half = mul(0.5, angle);
    double s, c;
    sincos(half, &s, &c);
    dq[0] = c;
    dq[1] = dv(mul(s, phi.x), angle);
    dq[2] = dv(mul(s, phi.y), angle);
    dq[3] = dv(mul(s, phi.z), angle);
  }
  qmul(dq, q, out);
  normalize4(out);
}

// quaternions.rotate (:42-51): v + 2 (w (u x v) + u x (u x v))
__device__ __forceinline__ V3 rotate(const double q[4], V3 v) {
  const V3 u{q[1], q[2], q[3]};
  const V3 uv = cross(u, v);
  const V3 inner = scale(uv, q[0]) + cross(u, uv);
  return v + scale(inner, 2.0);
}

// quaternions.to_matrix (:54-63), Python scalar arithmetic as written
__device__ __forceinline__ void to_matrix(const double q[4], double m[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  m[0] = sub(1.0, mul(2.0, add(mul(y, y), mul(z, z))));
  m[1] = mul(2.0, sub(mul(x, y), mul(w, z)));
  m[2] = mul(2.0, add(mul(x, z), mul(w, y)));
  m[3] = mul(2.0, add(mul(x, y), mul(w, z)));
  m[4] = sub(1.0, mul(2.0, add(mul(x, x), mul(z, z))));
  m[5] = mul(2.0, sub(mul(y, z), mul(w, x)));
  m[6] = mul(2.0, sub(mul(x, z), mul(w, y)));
  m[7] = mul(2.0, add(mul(y, z), mul(w, x)));
  m[8] = sub(1.0, mul(2.0, add(mul(x, x), mul(y, y))));
}

}  // namespace ltsg
