// Moving-path screen (dt > 0 batches: c4, c5), one generation as three
// kernels.  Included by search.cu after the candidate/record helpers.
//
//   k_mscreen  one warp per 32 frontier candidates: per candidate the
//              reference's sample count, grid and thresholds (ccd.py:321-370,
//              :410-411) and the certified window cull; per in-window row
//              (flattened over the warp's lanes) the moved-sphere cull and
//              the separating-axis cull.  The surviving rows are appended,
//              per warp and in candidate order, to a global row list.  No
//              exact distance here, so the kernel stays small and resident.
//   k_mexact   one thread per surviving row: the exact 15-feature distance
//              at the row's tau (pose table or Rodrigues, ccd.py:116-132)
//              and its three decision bits.
//   k_mdecide  one thread per row; the first row of each candidate's
//              segment gathers the candidate's bits and makes the
//              reference's decisions (ccd.py:404-446): resting record,
//              children of a flagged coarse candidate, flagged fine runs.
//              Rows settled by a cull carry no bits, exactly as a row whose
//              distance clears every threshold.
//
// Every tau is the reference's linspace sample; the per-candidate step is
// computed once (the same division linspace_at performs) and a row's tau is
// i*step + w0, bit for bit what linspace_at returns.

struct ExactRow {
  uint32_t cand;  // frontier index of the candidate
  int16_t i;      // sample index in linspace(w0, dt, count)
  uint8_t count;  // the candidate's sample count (1..33)
  uint8_t bits;   // k_mexact: 1 = flag (d <= thr), 2 = d <= h, 4 = resting test (d <= h + 1e-9)
  double tau;
  double thr;     // h + 0.5 * speed * step (ccd.py:410-411)
};
static_assert(sizeof(ExactRow) == 24, "ExactRow layout");

struct RowList {
  ExactRow* rows;
  unsigned long long cap;
  unsigned long long* n;  // device counter of this generation's rows
};

struct MCandInfo {
  double w0, dt, h, thr, step, cull_lo, cull_hi;
  int64_t off_a, off_b;  // record indices of the two triangles
  int32_t ba, bb, count, first, culled;
  int32_t tab;  // bit 0 / bit 1: the pose table covers side a / b
};

// linspace(w0, dt, count)[i] with the candidate's precomputed step
__device__ __forceinline__ double cand_tau(const MCandInfo& c, int i) {
  if (c.count <= 1) return c.w0;
  if (i == c.count - 1) return c.dt;
  if (c.step != 0.0) return add(mul((double)i, c.step), c.w0);
  return linspace_at(c.w0, c.dt, c.count, i);
}

#ifndef LTSG_PLANE_CULL
#define LTSG_PLANE_CULL 0  // measured: costs more than it saves
#endif
#ifndef LTSG_MSCREEN_MINB
#define LTSG_MSCREEN_MINB 5
#endif
#ifndef LTSG_MSCREEN_WARPS
#define LTSG_MSCREEN_WARPS 4
#endif
constexpr int kMWarps = LTSG_MSCREEN_WARPS;

// Per-candidate sphere-centre trajectory for the window and per-row sphere
// culls.  With the body's cull constants (k_cull_prep: x0, v, and the
// regrouped Rodrigues base / K base / K^2 base) a triangle's bounding-sphere
// centre s moves as
//   c(tau) = (x0 + base s) + tau v + sin(w tau) (K base s) + (1 - cos(w tau)) (K^2 base s),
// so the centre difference of the two triangles is 18 constants plus the
// two angular speeds; a row evaluates it from shared memory with two
// sincos and no rotation matrix.  The cull margin's scale uses a bound of
// |c| over [0, dt] (|x0 + base s| + dt |v| + |K base s| + 2 |K^2 base s|),
// so it never underestimates the per-row scale.
// Layout (SoA over the warp's 32 candidates): [0..2] dP0, [3..5] dV,
// [6..8] Ba, [9..11] Ca, [12..14] Bb, [15..17] Cb, [18] wa, [19] wb,
// [20] lim^2 of the row test (+inf: slivers are never culled), [21] scale bound.
constexpr int kTraj = 22;

struct TrajSide {
  double p0[3], v[3], b[3], c[3], w, bound;
};

__device__ __forceinline__ TrajSide traj_side(const double* cm, const double* r, double dt) {
  TrajSide t;
  const double x = __ldg(r + 12), y = __ldg(r + 13), z = __ldg(r + 14);
  const bool spin = __ldg(cm + 34) != 0.0;
  t.w = spin ? __ldg(cm + 33) : 0.0;
  t.bound = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    t.p0[k] = fma(__ldg(cm + 6 + 3 * k), x, fma(__ldg(cm + 7 + 3 * k), y, fma(__ldg(cm + 8 + 3 * k), z, __ldg(cm + k))));
    t.v[k] = __ldg(cm + 3 + k);
    t.b[k] = spin ? fma(__ldg(cm + 15 + 3 * k), x, fma(__ldg(cm + 16 + 3 * k), y, __ldg(cm + 17 + 3 * k) * z)) : 0.0;
    t.c[k] = spin ? fma(__ldg(cm + 24 + 3 * k), x, fma(__ldg(cm + 25 + 3 * k), y, __ldg(cm + 26 + 3 * k) * z)) : 0.0;
    t.bound += fabs(t.p0[k]) + dt * fabs(t.v[k]) + fabs(t.b[k]) + 2.0 * fabs(t.c[k]);
  }
  return t;
}

// squared centre distance at tau from a warp's trajectory table (candidate o)
__device__ __forceinline__ double traj_d2(const double (*tr)[32], int o, double tau) {
  double sa = 0.0, ca = 0.0, sb = 0.0, cb = 0.0;
  const double wa = tr[18][o], wb = tr[19][o];
  if (wa != 0.0) {
    sincos(wa * tau, &sa, &ca);
    ca = 1.0 - ca;
  }
  if (wb != 0.0) {
    sincos(wb * tau, &sb, &cb);
    cb = 1.0 - cb;
  }
  double d2 = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double d = fma(tau, tr[3 + k][o], tr[k][o]);
    d = fma(sa, tr[6 + k][o], d);
    d = fma(ca, tr[9 + k][o], d);
    d = fma(-sb, tr[12 + k][o], d);
    d = fma(-cb, tr[15 + k][o], d);
    d2 = fma(d, d, d2);
  }
  return d2;
}
// The same trajectory from registers: tr[0..2] dP0, [3..5] dV, [6..8] Ba,
// [9..11] Ca, [12..14] Bb, [15..17] Cb, [18] wa, [19] wb.
__device__ __forceinline__ double traj_d2_regs(const double* tr, double tau) {
  double sa = 0.0, ca = 0.0, sb = 0.0, cb = 0.0;
  if (tr[18] != 0.0) {
    sincos(tr[18] * tau, &sa, &ca);
    ca = 1.0 - ca;
  }
  if (tr[19] != 0.0) {
    sincos(tr[19] * tau, &sb, &cb);
    cb = 1.0 - cb;
  }
  double d2 = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double d = fma(tau, tr[3 + k], tr[k]);
    d = fma(sa, tr[6 + k], d);
    d = fma(ca, tr[9 + k], d);
    d = fma(-sb, tr[12 + k], d);
    d = fma(-cb, tr[15 + k], d);
    d2 = fma(d, d, d2);
  }
  return d2;
}

// A candidate's trajectory constants and the limit of its per-row sphere
// test (`lim`: radii + threshold + cull margin; +inf for slivers, which are
// never culled) and the coordinate scale the margins are taken from.
__device__ __forceinline__ void traj_build(const double* cma, const double* ra_, const double* cmb, const double* rb_,
                                           double dt, double thr, double h, double* tr, double* lim, double* scale) {
  const TrajSide sa_ = traj_side(cma, ra_, dt);
  const TrajSide sb_ = traj_side(cmb, rb_, dt);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    tr[k] = sa_.p0[k] - sb_.p0[k];
    tr[3 + k] = sa_.v[k] - sb_.v[k];
    tr[6 + k] = sa_.b[k];
    tr[9 + k] = sa_.c[k];
    tr[12 + k] = sb_.b[k];
    tr[15 + k] = sb_.c[k];
  }
  tr[18] = sa_.w;
  tr[19] = sb_.w;
  const double rA = __ldg(ra_ + 15), rB = __ldg(rb_ + 15);
  *scale = 1.0 + sa_.bound + sb_.bound + fabs(rA) + fabs(rB);
  const double T = fmax(thr, add(h, kRestSlop));
  *lim = (rA >= 0.0 && rB >= 0.0) ? rA + rB + T + kCullMargin * *scale : CUDART_INF;
}

#ifndef LTSG_MSCREEN_F32
#define LTSG_MSCREEN_F32 0  // FP32 pre-test of the per-row sphere cull, FP64 only inside its error band (measured: no gain)
#endif
// FP32 evaluation of the trajectory distance.  With s32 the sum of the
// magnitudes of the terms it adds (|dP0| + dt |dV| + |B| + 2 |C| per side,
// plus lim), its error against the FP64 value is below 4e-6 * s32
// (conversion of the 20 constants and of tau, ~20 roundings of partial sums
// bounded by s32, and the 4e-7 absolute error of __sincosf on |w tau| < pi
// times the rotation coefficients); the band below uses 1e-4 * s32, 25x that.  A row
// is settled in FP32 only when its distance clears the band on either side:
// culled above lim + E, kept below lim - E.  Rows inside the band take the
// FP64 test, so the surviving rows are exactly those of the FP64 test.
constexpr double kF32Band = 1e-4;
constexpr int kTrajF = 22;  // 18 constants, wa, wb, (lim + E)^2, (lim - E)^2

// the FP64 per-row sphere test from scratch (rows inside the FP32 band)
__device__ __noinline__ bool sphere_keep_f64(const double* cma, const double* ra_, const double* cmb,
                                             const double* rb_, double dt, double thr, double h, double tau) {
  double tr[20], lim, scale;
  traj_build(cma, ra_, cmb, rb_, dt, thr, h, tr, &lim, &scale);
  return !(traj_d2_regs(tr, tau) > lim * lim);
}

__device__ __forceinline__ float traj_d2f(const float (*tr)[32], int o, float tau) {
  float sa = 0.f, ca = 0.f, sb = 0.f, cb = 0.f;
  const float wa = tr[18][o], wb = tr[19][o];
  if (wa != 0.f) {
    __sincosf(wa * tau, &sa, &ca);
    ca = 1.f - ca;
  }
  if (wb != 0.f) {
    __sincosf(wb * tau, &sb, &cb);
    cb = 1.f - cb;
  }
  float d2 = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float d = __fmaf_rn(tau, tr[3 + k][o], tr[k][o]);
    d = __fmaf_rn(sa, tr[6 + k][o], d);
    d = __fmaf_rn(ca, tr[9 + k][o], d);
    d = __fmaf_rn(-sb, tr[12 + k][o], d);
    d = __fmaf_rn(-cb, tr[15 + k][o], d);
    d2 = __fmaf_rn(d, d, d2);
  }
  return d2;
}

constexpr int kMRows = 32 * kMaxSamples;  // rows of one warp's 32 candidates, at most

// Pose for the culls at sample i of linspace(w0, dt, n) (= tau): the pose
// table entry when the sample is on the body's table grid, else the
// regrouped Rodrigues rotation from the body's cull constants with sin/cos
// of w tau on the fly (fewer operations than the reference-rounded
// rotation_at; culls only, the margins cover the rounding).
__device__ __forceinline__ void mcull_pose(const BodyInfo* bodies, int b, double tau, bool use_tab, int n, int i,
                                           const PoseTable& pt, double R[9], double pos[3]) {
  if (pt.cm == nullptr || (use_tab && pt.tab != nullptr)) {
    // on the body's table grid the pose entry (6 vector loads) is cheaper
    // than the regrouped form (27 constants + 2 trig values)
    pose_at(bodies[b], b, tau, use_tab, n, i, pt, R, pos);
    return;
  }
  const double* cm = pt.cm + (size_t)b * kCullM;
#pragma unroll
  for (int k = 0; k < 3; ++k) pos[k] = fma(tau, __ldg(cm + 3 + k), __ldg(cm + k));
  if (__ldg(cm + 34) == 0.0) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(cm + 6 + k);
    return;
  }
  double sn, co;
  sincos(__ldg(cm + 33) * tau, &sn, &co);
  const double c = 1.0 - co;
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = fma(c, __ldg(cm + 24 + k), fma(sn, __ldg(cm + 15 + k), __ldg(cm + 6 + k)));
}

// Bounding-sphere gap at sample i (see sphere_gap_at), on the cull poses.
__device__ __forceinline__ double msphere_gap(const BodyInfo* bodies, int ba, int bb, const double* ra,
                                              const double* rb, double tau, int tab, int n, int i,
                                              const PoseTable& pt, double* scale) {
  double c[6];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const double* r = side ? rb : ra;
    double R[9], pos[3];
    mcull_pose(bodies, side ? bb : ba, tau, (tab >> side) & 1, n, i, pt, R, pos);
    const double x = __ldg(r + 12), y = __ldg(r + 13), z = __ldg(r + 14);
    c[3 * side] = fma(R[0], x, fma(R[1], y, fma(R[2], z, pos[0])));
    c[3 * side + 1] = fma(R[3], x, fma(R[4], y, fma(R[5], z, pos[1])));
    c[3 * side + 2] = fma(R[6], x, fma(R[7], y, fma(R[8], z, pos[2])));
  }
  const double dx = c[0] - c[3], dy = c[1] - c[4], dz = c[2] - c[5];
  const double rA = __ldg(ra + 15), rB = __ldg(rb + 15);
  *scale = 1.0 + fabs(c[0]) + fabs(c[1]) + fabs(c[2]) + fabs(c[3]) + fabs(c[4]) + fabs(c[5]) + rA + rB;
  return sqrt(fma(dx, dx, fma(dy, dy, dz * dz))) - (rA + rB);
}

// Separating-axis cull of one row (see sat_cull_posed), on the cull poses.
__device__ __forceinline__ bool msat_cull(const BodyInfo* bodies, int ba, int bb, const double* ra, const double* rb,
                                          double tau, int tab, int n, int i, const PoseTable& pt, double thr) {
  if (__ldg(ra + 15) < 0.0 || __ldg(rb + 15) < 0.0) return false;  // slivers are never culled
  double a[9], b[9];
  {
    double R[9], pos[3];
    mcull_pose(bodies, ba, tau, tab & 1, n, i, pt, R, pos);
    world_corners_fast(R, pos, ra, a);
    mcull_pose(bodies, bb, tau, (tab >> 1) & 1, n, i, pt, R, pos);
    world_corners_fast(R, pos, rb, b);
  }
  double scale = 1.0 + __ldg(ra + 15) + __ldg(rb + 15);
#pragma unroll
  for (int k = 0; k < 3; ++k) scale += fabs(a[k]) + fabs(b[k]);
  const double T = thr + kCullMargin * scale;
  auto normal_gap = [&](const double* x, const double* y) {  // x's face normal
    const double e1x = x[3] - x[0], e1y = x[4] - x[1], e1z = x[5] - x[2];
    const double e2x = x[6] - x[0], e2y = x[7] - x[1], e2z = x[8] - x[2];
    const double nx = fma(e1y, e2z, -e1z * e2y), ny = fma(e1z, e2x, -e1x * e2z), nz = fma(e1x, e2y, -e1y * e2x);
    const double len = sqrt(fma(nx, nx, fma(ny, ny, nz * nz)));
    return axis_gap(nx, ny, nz, x, y) - T * len;
  };
  if (normal_gap(a, b) > 0.0) return true;
  if (normal_gap(b, a) > 0.0) return true;
  const double ux = (b[0] + b[3] + b[6]) - (a[0] + a[3] + a[6]);
  const double uy = (b[1] + b[4] + b[7]) - (a[1] + a[4] + a[7]);
  const double uz = (b[2] + b[5] + b[8]) - (a[2] + a[5] + a[8]);
  const double len = sqrt(fma(ux, ux, fma(uy, uy, uz * uz)));
  return axis_gap(ux, uy, uz, a, b) > T * len;
}

// Per-row moved-sphere cull, without the square root: the bounding spheres
// of both triangles moved to tau (same rigid motion as the triangles) are
// certainly farther apart than T when |c_a - c_b|^2 > (r_a + r_b + T + m)^2,
// m the cull margin (cull arithmetic, FMA allowed).
__device__ __forceinline__ bool sphere_clear_at(const BodyInfo* bodies, int ba, int bb, const double* ra,
                                                const double* rb, double tau, int tab, int n, int i,
                                                const PoseTable& pt, double T) {
  double c[6];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int b = side ? bb : ba;
    const double* r = side ? rb : ra;
    double R[9], pos[3];
    mcull_pose(bodies, b, tau, (tab >> side) & 1, n, i, pt, R, pos);
    const double x = __ldg(r + 12), y = __ldg(r + 13), z = __ldg(r + 14);
    c[3 * side] = fma(R[0], x, fma(R[1], y, fma(R[2], z, pos[0])));
    c[3 * side + 1] = fma(R[3], x, fma(R[4], y, fma(R[5], z, pos[1])));
    c[3 * side + 2] = fma(R[6], x, fma(R[7], y, fma(R[8], z, pos[2])));
  }
  const double dx = c[0] - c[3], dy = c[1] - c[4], dz = c[2] - c[5];
  const double rr = __ldg(ra + 15) + __ldg(rb + 15);
  const double scale = 1.0 + fabs(c[0]) + fabs(c[1]) + fabs(c[2]) + fabs(c[3]) + fabs(c[4]) + fabs(c[5]) + rr;
  const double lim = rr + T + kCullMargin * scale;
  return fma(dx, dx, fma(dy, dy, dz * dz)) > lim * lim;
}

// Plane-sphere cull of one row: the plane of each triangle at tau against
// the other triangle's moved bounding sphere.  The triangle lies in its
// plane, so a sphere entirely on one side by more than T + m certifies a
// distance above T.  Body-frame normal from the record's corners (rotation
// keeps |n| and n . v0), so only R n and n . pos are per row; compared in
// squares, no square root (cull arithmetic, FMA allowed).
__device__ __forceinline__ bool plane_sphere_clear(const BodyInfo* bodies, int ba, int bb, const double* ra,
                                                   const double* rb, double tau, int tab, int n, int i,
                                                   const PoseTable& pt, double T) {
  double c[6], Rs[2][9], ps[2][3];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int b = side ? bb : ba;
    const double* r = side ? rb : ra;
    mcull_pose(bodies, b, tau, (tab >> side) & 1, n, i, pt, Rs[side], ps[side]);
    const double* R = Rs[side];
    const double x = __ldg(r + 12), y = __ldg(r + 13), z = __ldg(r + 14);
    c[3 * side] = fma(R[0], x, fma(R[1], y, fma(R[2], z, ps[side][0])));
    c[3 * side + 1] = fma(R[3], x, fma(R[4], y, fma(R[5], z, ps[side][1])));
    c[3 * side + 2] = fma(R[6], x, fma(R[7], y, fma(R[8], z, ps[side][2])));
  }
  const double scale = 1.0 + fabs(c[0]) + fabs(c[1]) + fabs(c[2]) + fabs(c[3]) + fabs(c[4]) + fabs(c[5]) +
                       __ldg(ra + 15) + __ldg(rb + 15);
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const double* r = side ? rb : ra;    // the plane's triangle
    const double* q = side ? c : c + 3;  // the other sphere's centre
    const double rad = __ldg((side ? ra : rb) + 15);
    const double* R = Rs[side];
    const double v0x = __ldg(r), v0y = __ldg(r + 1), v0z = __ldg(r + 2);
    const double e1x = __ldg(r + 3) - v0x, e1y = __ldg(r + 4) - v0y, e1z = __ldg(r + 5) - v0z;
    const double e2x = __ldg(r + 6) - v0x, e2y = __ldg(r + 7) - v0y, e2z = __ldg(r + 8) - v0z;
    const double lx = fma(e1y, e2z, -e1z * e2y), ly = fma(e1z, e2x, -e1x * e2z), lz = fma(e1x, e2y, -e1y * e2x);
    const double nx = fma(R[0], lx, fma(R[1], ly, R[2] * lz));
    const double ny = fma(R[3], lx, fma(R[4], ly, R[5] * lz));
    const double nz = fma(R[6], lx, fma(R[7], ly, R[8] * lz));
    // n . (x - (R v0 + pos)) = n . x - (l . v0 + n . pos)
    const double o = fma(lx, v0x, fma(ly, v0y, lz * v0z)) + fma(nx, ps[side][0], fma(ny, ps[side][1], nz * ps[side][2]));
    const double dist_n = fma(nx, q[0], fma(ny, q[1], nz * q[2])) - o;  // signed distance times |n|
    const double lim = rad + T + kCullMargin * scale;
    if (lim > 0.0 && dist_n * dist_n > lim * lim * fma(lx, lx, fma(ly, ly, lz * lz))) return true;
  }
  return false;
}

__device__ __forceinline__ int owner_of(const MCandInfo* info, int r) {
  int o = 0;  // last lane with first <= r among lanes that own rows
#pragma unroll
  for (int step = 16; step > 0; step >>= 1)
    if (info[o + step].first <= r) o += step;
  while (info[o].culled || info[o].count == 0) --o;
  return o;
}

__global__ void __launch_bounds__(32 * kMWarps, LTSG_MSCREEN_MINB)
k_mscreen(const Cand* __restrict__ front, int64_t n, const PairInfo* __restrict__ pairs,
          const BodyInfo* __restrict__ bodies, const double* __restrict__ tris, ScreenOut out, PoseTable pt,
          RowList rl) {
  if (out.n_in) n = (int64_t)min(*out.n_in, out.next_cap);
  __shared__ MCandInfo s_info[kMWarps][32];
  __shared__ uint16_t s_queue[kMWarps][kMRows];  // row (11 bits) | owner lane << 11
#if LTSG_MSCREEN_F32
  __shared__ float s_traj[kMWarps][kTrajF][32];
#else
  __shared__ double s_traj[kMWarps][kTraj][32];
#endif
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (n + 31) / 32;
  MCandInfo* info = s_info[warp];
  uint16_t* queue = s_queue[warp];
#if LTSG_MSCREEN_F32
  float(*traj)[32] = s_traj[warp];
#else
  double(*traj)[32] = s_traj[warp];
#endif
  unsigned long long acc_rows = 0, acc_exact = 0, acc_window = 0, acc_sphere = 0;

  for (int64_t wi = blockIdx.x * (int64_t)kMWarps + warp; wi < n_warps; wi += (int64_t)gridDim.x * kMWarps) {
    const int64_t ci = wi * 32 + lane;
    MCandInfo me{};
    if (ci < n) {
      const Cand c = front[ci];
      const PairInfo p = pairs[c.pair];
      const BodyInfo& A = bodies[p.ba];
      const BodyInfo& B = bodies[p.bb];
      me.ba = p.ba;
      me.bb = p.bb;
      me.off_a = A.level_off[c.la] + c.ia;
      me.off_b = B.level_off[c.lb] + c.ib;
      const double* ra_ = tris + me.off_a * kRecord;
      const double* rb_ = tris + me.off_b * kRecord;
      me.h = add(__ldg(ra_ + 9), __ldg(rb_ + 9));  // ccd.py:339
      double sp = p.speed0;                        // ccd.py:340-345
      if (A.m.omega > 0.0) sp = add(sp, mul(A.m.omega, __ldg(ra_ + 10)));
      if (B.m.omega > 0.0) sp = add(sp, mul(B.m.omega, __ldg(rb_ + 10)));
      me.w0 = c.w0;
      me.tab = (pt.tab != nullptr && c.w0 == 0.0)
          ? ((pt.tdt[p.ba] == p.dt ? 1 : 0) | (pt.tdt[p.bb] == p.dt ? 2 : 0)) : 0;
      me.dt = p.dt;
      const double span = fmax(sub(p.dt, c.w0), 0.0);
      me.count = sample_count(span, sp, me.h);
      // linspace's step, once (numpy: (stop - start) / (n - 1))
      me.step = me.count > 1 ? dv(sub(p.dt, c.w0), (double)(me.count - 1)) : 0.0;
      const double step = me.count > 1 ? sub(cand_tau(me, 1), c.w0) : 0.0;  // grid[1] - grid[0]
      me.thr = add(me.h, mul(mul(0.5, sp), step));  // ccd.py:410-411
      // certified window (see k_screen): the bounding-sphere gap is
      // `speed`-Lipschitz, evaluated at both window ends
      me.cull_lo = -1.0;
      me.cull_hi = 2.0 * p.dt + 1.0;
      // the sphere-centre trajectories (see kTraj)
      double tr[20], lim, scale;
      traj_build(pt.cm + (size_t)p.ba * kCullM, ra_, pt.cm + (size_t)p.bb * kCullM, rb_, p.dt, me.thr, me.h, tr, &lim,
                 &scale);
#if LTSG_MSCREEN_F32
#pragma unroll
      for (int k = 0; k < 20; ++k) traj[k][lane] = (float)tr[k];
      {
        // the magnitudes the FP32 evaluation actually handles: the centre
        // DIFFERENCE and its rates (not the absolute positions in `scale`)
        double s32 = lim < CUDART_INF ? lim : 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          s32 += fabs(tr[k]) + p.dt * fabs(tr[3 + k]) + fabs(tr[6 + k]) + 2.0 * fabs(tr[9 + k]) + fabs(tr[12 + k]) +
                 2.0 * fabs(tr[15 + k]);
        const double E = kF32Band * s32;
        const double hi = lim + E, lo = fmax(lim - E, 0.0);
        // rounded outwards, so the FP32 limits never narrow the band
        traj[20][lane] = lim < CUDART_INF ? __double2float_ru(hi * hi) : CUDART_INF_F;
        traj[21][lane] = lim < CUDART_INF ? __double2float_rd(lo * lo) : CUDART_INF_F;
        if (!(s32 < 1e15) && lim < CUDART_INF) {  // beyond a safe FP32 range: every row takes the FP64 test
          traj[20][lane] = CUDART_INF_F;
          traj[21][lane] = 0.f;
        }
      }
#else
#pragma unroll
      for (int k = 0; k < 20; ++k) traj[k][lane] = tr[k];
      traj[20][lane] = lim < CUDART_INF ? lim * lim : CUDART_INF;
#endif
      if (lim < CUDART_INF) {
        const double g0 = sqrt(traj_d2_regs(tr, c.w0)) - lim;
        double g1 = g0;
        if (p.dt > c.w0) g1 = sqrt(traj_d2_regs(tr, p.dt)) - lim;
        if (sp > 0.0) {
          me.cull_lo = c.w0 + g0 / sp;
          me.cull_hi = p.dt - g1 / sp;
        } else if (g0 > 0.0) {
          me.cull_lo = 2.0 * p.dt + 1.0;
        }
        me.culled = me.cull_lo > p.dt || me.cull_hi < c.w0 || me.cull_lo > me.cull_hi;
      }
    }
    const int nrows = me.culled ? 0 : me.count;
    const int incl = warp_incl_scan(nrows, lane);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int all_rows = me.count;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) all_rows += __shfl_xor_sync(0xffffffffu, all_rows, o);
    me.first = incl - nrows;
    info[lane] = me;
    __syncwarp();

    // (a) window + moved-sphere cull per row; survivors queued with their owner
    int nq = 0;
    for (int r0 = 0; r0 < total; r0 += 32) {
      const int r = r0 + lane;
      bool keep = false;
      int o = 0;
      if (r < total) {
        o = owner_of(info, r);
        const MCandInfo& c = info[o];
        const int i = r - c.first;
        const double tau = cand_tau(c, i);
        keep = !(tau < c.cull_lo || tau > c.cull_hi);
#if LTSG_MSCREEN_F32
        if (keep) {
          const float d2f = traj_d2f(traj, o, (float)tau);
          if (d2f > traj[20][o]) {
            keep = false;  // certainly clear
          } else if (!(d2f < traj[21][o])) {
            // inside the FP32 error band: the FP64 test decides
            keep = sphere_keep_f64(pt.cm + (size_t)c.ba * kCullM, tris + c.off_a * kRecord,
                                   pt.cm + (size_t)c.bb * kCullM, tris + c.off_b * kRecord, c.dt, c.thr, c.h, tau);
          }
        }
#else
        if (keep) keep = !(traj_d2(traj, o, tau) > traj[20][o]);
#endif
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) queue[nq + __popc(m & ((1u << lane) - 1u))] = (uint16_t)(r | (o << 11));
      nq += __popc(m);
    }
    __syncwarp();
    const int nq_sphere = nq;
#if LTSG_PLANE_CULL
    // (b0) plane-sphere cull of the sphere survivors, compacted in place
    {
      int nq2 = 0;
      for (int q0 = 0; q0 < nq; q0 += 32) {
        const int q = q0 + lane;
        bool keep = false;
        uint16_t e = 0;
        if (q < nq) {
          e = queue[q];
          const int r = e & 2047, o = e >> 11;
          const MCandInfo& c = info[o];
          const int i = r - c.first;
          keep = !plane_sphere_clear(bodies, c.ba, c.bb, tris + c.off_a * kRecord, tris + c.off_b * kRecord,
                                     cand_tau(c, i), c.tab, c.count, i, pt, fmax(c.thr, add(c.h, kRestSlop)));
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) queue[nq2 + __popc(m & ((1u << lane) - 1u))] = e;
        nq2 += __popc(m);
      }
      nq = nq2;
    }
    __syncwarp();
#endif
    // (b) separating-axis cull of the sphere survivors, compacted in place
    {
      int nq2 = 0;
      for (int q0 = 0; q0 < nq; q0 += 32) {
        const int q = q0 + lane;
        bool keep = false;
        uint16_t e = 0;
        if (q < nq) {
          e = queue[q];
          const int r = e & 2047, o = e >> 11;
          const MCandInfo& c = info[o];
          const int i = r - c.first;
          keep = !msat_cull(bodies, c.ba, c.bb, tris + c.off_a * kRecord, tris + c.off_b * kRecord,
                            cand_tau(c, i), c.tab, c.count, i, pt, fmax(c.thr, add(c.h, kRestSlop)));
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) queue[nq2 + __popc(m & ((1u << lane) - 1u))] = e;
        nq2 += __popc(m);
      }
      nq = nq2;
    }
    __syncwarp();
    // (c) the survivors go to the global row list, in candidate order
    unsigned long long base = 0;
    if (lane == 0 && nq) base = atomicAdd(rl.n, (unsigned long long)nq);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int q = lane; q < nq; q += 32) {
      const uint16_t e = queue[q];
      const int r = e & 2047, o = e >> 11;
      const MCandInfo& c = info[o];
      const int i = r - c.first;
      const unsigned long long dst = base + q;
      if (dst < rl.cap) {
        ExactRow x;
        x.cand = (uint32_t)(wi * 32 + o);
        x.i = (int16_t)i;
        x.count = (uint8_t)c.count;
        x.bits = 0;
        x.tau = cand_tau(c, i);
        x.thr = c.thr;
        rl.rows[dst] = x;
      }
    }
    acc_rows += (unsigned long long)all_rows;
    acc_exact += (unsigned long long)nq;
    acc_window += (unsigned long long)total;
    acc_sphere += (unsigned long long)nq_sphere;
    __syncwarp();
  }
  if (lane == 0) {
    if (acc_rows) atomicAdd(&out.ctr->rows, acc_rows);
    if (acc_exact) atomicAdd(&out.ctr->screen_exact, acc_exact);
    if (acc_window) atomicAdd(&out.ctr->rows_window, acc_window);
    if (acc_sphere) atomicAdd(&out.ctr->rows_sphere, acc_sphere);
  }
}

#ifndef LTSG_MEXACT_MINB
#define LTSG_MEXACT_MINB 7
#endif
constexpr int kMExactThreads = 128;
constexpr int kMExactWarps = kMExactThreads / 32;
constexpr int kMExactStageBytes = kStagedLite * kMExactThreads * sizeof(double);

// World triangles of a row's two records at the row's tau (pose table or
// Rodrigues, the reference's rounding).
__device__ __forceinline__ void row_world(const BodyInfo* bodies, int ba, int bb, const double* ra, const double* rb,
                                          double tau, int tab, int n, int i, const PoseTable& pt, Tri* ta, Tri* tb) {
  {
    double R[9], pos[3], L[9];
    pose_at(bodies[ba], ba, tau, tab & 1, n, i, pt, R, pos);
    load_local(ra, L);
    *ta = world_tri(R, pos, L);
  }
  {
    double R[9], pos[3], L[9];
    pose_at(bodies[bb], bb, tau, (tab >> 1) & 1, n, i, pt, R, pos);
    load_local(rb, L);
    *tb = world_tri(R, pos, L);
  }
}

struct MRowCtx {
  const double *ra, *rb;
  double h;
  int ba, bb, tab;
};

__device__ __forceinline__ MRowCtx mrow_ctx(const ExactRow& r, const Cand* front, const PairInfo* pairs,
                                            const BodyInfo* bodies, const double* tris, const PoseTable& pt) {
  const Cand c = front[r.cand];
  const PairInfo p = pairs[c.pair];
  MRowCtx x;
  x.ba = p.ba;
  x.bb = p.bb;
  x.ra = tris + (bodies[p.ba].level_off[c.la] + c.ia) * kRecord;
  x.rb = tris + (bodies[p.bb].level_off[c.lb] + c.ib) * kRecord;
  x.h = add(__ldg(x.ra + 9), __ldg(x.rb + 9));
  x.tab = (pt.tab != nullptr && c.w0 == 0.0) ? ((pt.tdt[p.ba] == p.dt ? 1 : 0) | (pt.tdt[p.bb] == p.dt ? 2 : 0)) : 0;
  return x;
}

// The rows' three decision bits (1 = flag d <= thr, 2 = d <= h, 4 = resting
// test d <= h + 1e-9).  Pass 1: the certified FP32 upper bound
// (bound32.cuh) decides rows certainly at or below their thresholds -- all
// three bits when the bound clears h; the flag alone for a sample i > 0
// (k_mdecide reads the touch and resting bits of sample 0 only, and of no
// flagged sample but the first).  Pass 2: the rows left undecided are
// queued per warp and evaluated with the bit-exact 15-feature distance, 32
// at a time, so the exact batches stay dense.
__global__ void __launch_bounds__(kMExactThreads, LTSG_MEXACT_MINB)
k_mexact(const Cand* __restrict__ front, const PairInfo* __restrict__ pairs, const BodyInfo* __restrict__ bodies,
         const double* __restrict__ tris, PoseTable pt, RowList rl, unsigned long long* n_bound) {
  extern __shared__ double s_stage[];
  __shared__ int64_t s_q[kMExactWarps][64];
  const Staged<kMExactThreads> st{s_stage + threadIdx.x};
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int64_t* q = s_q[warp];
  const int64_t n = (int64_t)min(*rl.n, rl.cap);
  const int64_t n_warps = (n + 31) / 32;
  int nq = 0;
  unsigned long long decided = 0;
  auto exact = [&](int64_t x) {
    const ExactRow r = rl.rows[x];
    const MRowCtx c = mrow_ctx(r, front, pairs, bodies, tris, pt);
    const double d = row_distance_posed(st, bodies, c.ba, c.bb, c.ra, c.rb, r.tau, c.tab, r.count, r.i, pt);
    uint8_t b = 0;
    if (d <= r.thr) b |= 1;
    if (d <= c.h) b |= 2;
    if (d <= add(c.h, kRestSlop)) b |= 4;
    rl.rows[x].bits = b;
  };
  for (int64_t wi = blockIdx.x * (int64_t)kMExactWarps + warp; wi < n_warps; wi += (int64_t)gridDim.x * kMExactWarps) {
    const int64_t x = wi * 32 + lane;
    bool pend = false;
    if (x < n) {
      const ExactRow r = rl.rows[x];
      const MRowCtx c = mrow_ctx(r, front, pairs, bodies, tris, pt);
      pend = true;
      if (LTSG_BOUND && __ldg(c.ra + 15) >= 0.0 && __ldg(c.rb + 15) >= 0.0) {
        Tri ta, tb;
        row_world(bodies, c.ba, c.bb, c.ra, c.rb, r.tau, c.tab, r.count, r.i, pt, &ta, &tb);
        double ub, margin;
        if (feature_ub(ta, tb, &ub, &margin)) {
          const double u = ub + margin;
          if (u <= c.h) {
            rl.rows[x].bits = 7;
            pend = false;
          } else if (r.i > 0 && u <= r.thr) {
            rl.rows[x].bits = 1;
            pend = false;
          }
        }
      }
      decided += !pend;
    }
    const unsigned m = __ballot_sync(0xffffffffu, pend);
    if (pend) q[nq + __popc(m & ((1u << lane) - 1u))] = x;
    nq += __popc(m);
    __syncwarp();
    if (nq >= 32) {
      exact(q[lane]);
      __syncwarp();
      if (lane < nq - 32) q[lane] = q[32 + lane];
      nq -= 32;
      __syncwarp();
    }
  }
  if (lane < nq) exact(q[lane]);
  for (int o = 16; o > 0; o >>= 1) decided += __shfl_xor_sync(0xffffffffu, decided, o);
  if (lane == 0 && decided) atomicAdd(n_bound, decided);
}

struct MChild {
  double w0;
  int32_t first, count, pair, ia0, ib0, nb, la, lb;
};

constexpr int kMDecideWarps = 8;

// Decisions per candidate (ccd.py:404-446) from its rows' bits.  The rows of
// one candidate are contiguous in the list; the first one of each segment
// acts.  Children of flagged coarse candidates are emitted warp-cooperatively
// (one atomic per warp, coalesced stores).
__global__ void __launch_bounds__(32 * kMDecideWarps)
k_mdecide(const Cand* __restrict__ front, const PairInfo* __restrict__ pairs, const BodyInfo* __restrict__ bodies,
          const double* __restrict__ tris, RowList rl, ScreenOut out) {
  __shared__ MChild s_kid[kMDecideWarps][32];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  MChild* kid = s_kid[warp];
  const int64_t n = (int64_t)min(*rl.n, rl.cap);
  const int64_t n_warps = (n + 31) / 32;
  for (int64_t wi = blockIdx.x * (int64_t)kMDecideWarps + warp; wi < n_warps;
       wi += (int64_t)gridDim.x * kMDecideWarps) {
    const int64_t x = wi * 32 + lane;
    MChild ch{};
    if (x < n) {
      const ExactRow r = rl.rows[x];
      const bool head = x == 0 || rl.rows[x - 1].cand != r.cand;
      uint64_t flag = 0, touch = 0;
      bool rest0 = false;
      if (head) {
        for (int64_t j = x; j < n; ++j) {
          const ExactRow s = rl.rows[j];
          if (s.cand != r.cand) break;
          if (s.bits & 1) flag |= 1ull << s.i;
          if (s.bits & 2) touch |= 1ull << s.i;
          if (s.i == 0 && (s.bits & 4)) rest0 = true;
        }
      }
      if (flag || rest0) {
        const Cand own = front[r.cand];
        const PairInfo p = pairs[own.pair];
        const BodyInfo& A = bodies[p.ba];
        const BodyInfo& B = bodies[p.bb];
        const int64_t off_a = A.level_off[own.la] + own.ia;
        const int64_t off_b = B.level_off[own.lb] + own.ib;
        const double* ra = tris + off_a * kRecord;
        const double* rb = tris + off_b * kRecord;
        const double h = add(__ldg(ra + 9), __ldg(rb + 9));
        const int count = r.count;
        const bool fine = own.la == 0 && own.lb == 0;
        if (fine && own.w0 == 0.0 && rest0) {
          const unsigned long long slot = atomicAdd(&out.ctr->resting, 1ULL);
          if (slot < out.rest_cap) out.resting[slot] = RestRec{own.pair, own.ia, own.ib, 0, h};
        } else if (flag && !fine) {  // ccd.py:414-428
          const int k0 = __ffsll((long long)flag) - 1;
          ch.w0 = linspace_at(own.w0, p.dt, count, k0 > 0 ? k0 - 1 : 0);
          ch.pair = own.pair;
          int na = 1, nb = 1;
          ch.ia0 = own.ia;
          ch.ib0 = own.ib;
          if (own.la > 0) {
            const int2 cr = *reinterpret_cast<const int2*>(ra + 11);
            ch.ia0 = cr.x;
            na = cr.y;
          }
          if (own.lb > 0) {
            const int2 cr = *reinterpret_cast<const int2*>(rb + 11);
            ch.ib0 = cr.x;
            nb = cr.y;
          }
          ch.nb = nb;
          ch.count = na * nb;
          ch.la = own.la > 0 ? own.la - 1 : 0;
          ch.lb = own.lb > 0 ? own.lb - 1 : 0;
        } else if (flag) {  // fine: flagged runs (ccd.py:429-446)
          double sp = p.speed0;
          if (A.m.omega > 0.0) sp = add(sp, mul(A.m.omega, __ldg(ra + 10)));
          if (B.m.omega > 0.0) sp = add(sp, mul(B.m.omega, __ldg(rb + 10)));
          int k = __ffsll((long long)flag) - 1;
          while (k < count) {
            if (!((flag >> k) & 1)) { ++k; continue; }
            int ke = k;
            while (ke + 1 < count && ((flag >> (ke + 1)) & 1)) ++ke;
            const int lo_i = k > 0 ? k - 1 : 0;
            const int hi_i = ke + 1 < count - 1 ? ke + 1 : count - 1;
            if ((touch >> lo_i) & 1) {
              const unsigned long long slot = atomicAdd(&out.ctr->cross, 1ULL);
              if (slot < out.cross_cap)
                out.cross[slot] = Cross{own.pair, own.ia, own.ib, 0, linspace_at(own.w0, p.dt, count, lo_i), h};
            } else if (hi_i > lo_i) {
              const unsigned long long slot = atomicAdd(&out.ctr->entries, 1ULL);
              if (slot < out.entry_cap)
                out.entries[slot] = Entry{own.pair, own.ia, own.ib, 0, linspace_at(own.w0, p.dt, count, lo_i),
                                          linspace_at(own.w0, p.dt, count, hi_i), h, sp};
            }
            k = ke + 1;
          }
        }
      }
    }
    // cooperative, coalesced child emission
    const int cincl = warp_incl_scan(ch.count, lane);
    const int ctotal = __shfl_sync(0xffffffffu, cincl, 31);
    if (ctotal) {
      unsigned long long cbase = 0;
      if (lane == 0) cbase = atomicAdd(out.n_out, (unsigned long long)ctotal);
      cbase = __shfl_sync(0xffffffffu, cbase, 0);
      ch.first = cincl - ch.count;
      kid[lane] = ch;
      __syncwarp();
      for (int s = lane; s < ctotal; s += 32) {
        int o = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (kid[o + step].first <= s) o += step;
        const MChild& c = kid[o];
        const int j = s - c.first;
        const unsigned long long dst = cbase + s;
        if (dst < out.next_cap) {
          Cand nc;
          nc.pair = c.pair;
          nc.ia = c.ia0 + j / c.nb;
          nc.ib = c.ib0 + j % c.nb;
          nc.la = (int16_t)c.la;
          nc.lb = (int16_t)c.lb;
          nc.w0 = c.w0;
          out.next[dst] = nc;
        }
      }
      __syncwarp();
    }
  }
}
