// Batched multiscale earliest-contact search: ccd._search (ccd.py:373-487)
// over many independent problems in one pass, plus contact records
// (ccd.py:183-213) and fusion (ccd.py:527-577).
//
// Schedule.  In the reference the fine (0,0) bucket is processed last and
// exactly once (bucket key max(la,lb) strictly decreases from parent to
// child, ccd.py:394 / 418-427), so the shared bound equals dt for the whole
// coarse traversal and the prune filters at ccd.py:396-397 / 448-449 never
// fire.  Every candidate is therefore screened over [w0, dt] independently
// of every other, and the traversal is an order-free frontier expansion.
// We run it level-synchronously over all problems at once ("generations"):
// the screen kernel evaluates every candidate of the frontier, expands the
// flagged coarse ones into the next frontier and turns fine ones into
// resting records, defensive crossings and refinement entries.  Zoom and
// bisection then run per entry; the bound of a problem is the minimum
// bisected tau (ccd.py:459-468), which is exactly what the reference's
// sorted narrowing loop produces.
#include "common.cuh"
#include "geom.cuh"
#include "dist_staged.cuh"
#include "dist_tile.cuh"

#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <ctime>
#include <vector>

#ifndef LTSG_BOUND
#define LTSG_BOUND 0  // certified FP32 upper-bound pre-decision in the exact kernels (measured: no net gain)
#endif

namespace ltsg {

constexpr int kMaxLevels = 8;
constexpr int kRecord = 16;  // doubles per triangle record
constexpr int kWorld = 20;   // doubles per tau = 0 world record
constexpr int kSph = 4;      // doubles per compact cull sphere (after the world records)
// Relative slack of the certified culls: rows within this (times the
// coordinate scale) of a threshold are always evaluated exactly.
constexpr double kCullMargin = 1e-7;
// slivers (Lmax^2 > 1e4 |e0 x e2|, packing.CULL_COND) carry radius -1 and are never culled
}  // namespace ltsg
#include "bound32.cuh"
namespace ltsg {

struct BodyInfo {
  Motion m;
  int64_t level_off[kMaxLevels];
  int32_t level_size[kMaxLevels];
  int32_t n_levels;
  int32_t id;
};

struct PairInfo {
  int32_t ba, bb, problem, group;
  double speed0;  // |v_a - v_b| (ddot norm)
  double dt;
};

struct Cand {
  int32_t pair;
  int32_t ia;  // level-local record index (children contiguous)
  int32_t ib;
  int16_t la, lb;
  double w0;
};
static_assert(sizeof(Cand) == 24, "Cand layout");

struct RestRec {
  int32_t pair, ia, ib, pad;
  double h;
};
struct Entry {
  int32_t pair, ia, ib, pad;
  double lo, hi, h, speed;
};
struct Cross {
  int32_t pair, ia, ib, pad;
  double tau, h;
};
struct Bracket {
  int32_t pair, ia, ib, pad;
  double lo, hi, h;
};

struct Counters {
  unsigned long long next;       // next-frontier size
  unsigned long long resting;
  unsigned long long entries;
  unsigned long long cross;
  unsigned long long rows;       // screen rows (reference-equivalent)
  unsigned long long brackets;
  unsigned long long zoom_rows;  // rows the reference would evaluate
  unsigned long long zoom_exec;  // rows evaluated here
  unsigned long long bisect_rows;
  unsigned long long records;
  unsigned long long overflow;   // zoom queue overflow flag
  unsigned long long screen_exact;  // screen rows evaluated with the exact 15-feature distance
  unsigned long long rows_window;   // moving screen: rows inside the candidates' cull windows
  unsigned long long rows_sphere;   // moving screen: rows surviving the per-row sphere cull
  unsigned long long bound_rows;    // screen_exact rows decided by the certified FP32 upper bound
};

// ---------------------------------------------------------------- prep

__global__ void k_prep_bodies(const double* state, const int64_t* levels, int n, BodyInfo* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = state + 16 * i;
  const int64_t* L = levels + 18 * i;
  BodyInfo b;
  b.n_levels = (int32_t)L[0];
  b.id = (int32_t)L[1];
  for (int l = 0; l < kMaxLevels; ++l) {
    b.level_off[l] = L[2 + l];
    b.level_size[l] = (int32_t)L[10 + l];
  }
  Motion& m = b.m;
  const bool is_static = s[13] != 0.0;
  if (is_static) {  // ccd.py:106: zero motion, identity pose
    for (int k = 0; k < 3; ++k) m.x0[k] = m.v[k] = 0.0;
    for (int k = 0; k < 9; ++k) m.base[k] = (k % 4 == 0) ? 1.0 : 0.0;
    m.omega = 0.0;
    m.spinning = 0;
  } else {
    for (int k = 0; k < 3; ++k) {
      m.x0[k] = s[k];
      m.v[k] = s[3 + k];
    }
    const double w = s[6], x = s[7], y = s[8], z = s[9];  // quaternions.to_matrix
    m.base[0] = sub(1.0, mul(2.0, add(mul(y, y), mul(z, z))));
    m.base[1] = mul(2.0, sub(mul(x, y), mul(w, z)));
    m.base[2] = mul(2.0, add(mul(x, z), mul(w, y)));
    m.base[3] = mul(2.0, add(mul(x, y), mul(w, z)));
    m.base[4] = sub(1.0, mul(2.0, add(mul(x, x), mul(z, z))));
    m.base[5] = mul(2.0, sub(mul(y, z), mul(w, x)));
    m.base[6] = mul(2.0, sub(mul(x, z), mul(w, y)));
    m.base[7] = mul(2.0, add(mul(y, z), mul(w, x)));
    m.base[8] = sub(1.0, mul(2.0, add(mul(x, x), mul(y, y))));
    const V3 om{s[10], s[11], s[12]};
    m.omega = norm_blas(om);
    m.spinning = m.omega > 0.0;
  }
  for (int k = 0; k < 9; ++k) m.K[k] = m.KK[k] = 0.0;
  if (m.spinning) {
    const double k0 = dv(s[10], m.omega), k1 = dv(s[11], m.omega), k2 = dv(s[12], m.omega);
    const double K[9] = {0.0, -k2, k1, k2, 0.0, -k0, -k1, k0, 0.0};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        m.K[3 * r + c] = K[3 * r + c];
        m.KK[3 * r + c] = fma_(K[3 * r + 2], K[6 + c], fma_(K[3 * r + 1], K[3 + c], mul(K[3 * r], K[c])));
      }
  }
  m.pad = 0;
  out[i] = b;
}

__global__ void k_prep_pairs(const int32_t* pair_body, const int32_t* pair_problem,
                             const int32_t* pair_group, int64_t n, const BodyInfo* bodies,
                             const double* problem_dt, PairInfo* out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  PairInfo p;
  p.ba = pair_body[2 * k];
  p.bb = pair_body[2 * k + 1];
  p.problem = pair_problem[k];
  p.group = pair_group[k];
  const Motion& a = bodies[p.ba].m;
  const Motion& b = bodies[p.bb].m;
  p.speed0 = norm_blas(V3{sub(a.v[0], b.v[0]), sub(a.v[1], b.v[1]), sub(a.v[2], b.v[2])});
  p.dt = problem_dt[p.problem];
  out[k] = p;
}

// ---------------------------------------------------------------- seeds

__device__ __forceinline__ void seed_levels(const PairInfo& p, const BodyInfo* bodies, int exhaustive,
                                            int* la, int* lb, int64_t* na, int64_t* nb) {
  const BodyInfo& A = bodies[p.ba];
  const BodyInfo& B = bodies[p.bb];
  *la = exhaustive ? 0 : A.n_levels - 1;
  *lb = exhaustive ? 0 : B.n_levels - 1;
  *na = A.level_size[*la];
  *nb = B.level_size[*lb];
}

__global__ void k_seed_count(const PairInfo* pairs, int64_t n, const BodyInfo* bodies, int exhaustive,
                             int64_t* count) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int la, lb;
  int64_t na, nb;
  seed_levels(pairs[k], bodies, exhaustive, &la, &lb, &na, &nb);
  count[k] = na * nb;
}

__global__ void k_seed_fill(const PairInfo* pairs, int64_t n, const BodyInfo* bodies, int exhaustive,
                            const int64_t* offset, Cand* out) {
  for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
    int la, lb;
    int64_t na, nb;
    seed_levels(pairs[k], bodies, exhaustive, &la, &lb, &na, &nb);
    const int64_t base = offset[k];
    for (int64_t j = threadIdx.x; j < na * nb; j += blockDim.x) {
      Cand c;
      c.pair = (int32_t)k;
      c.ia = (int32_t)(j / nb);
      c.ib = (int32_t)(j % nb);
      c.la = (int16_t)la;
      c.lb = (int16_t)lb;
      c.w0 = 0.0;
      out[base + j] = c;
    }
  }
}

// ---------------------------------------------------------------- rows

__device__ __forceinline__ const double* rec(const double* tris, const BodyInfo& b, int level, int idx) {
  return tris + (size_t)(b.level_off[level] + idx) * kRecord;
}

__device__ __forceinline__ void load_local(const double* r, double L[9]) {
  const double2* q = reinterpret_cast<const double2*>(r);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 t = __ldg(q + k);
    L[2 * k] = t.x;
    L[2 * k + 1] = t.y;
  }
  L[8] = __ldg(r + 8);
}

// World triangle of body record `r` at time tau.
__device__ __forceinline__ Tri world_at(const Motion& m, const double* r, double tau) {
  double L[9], R[9], pos[3];
  load_local(r, L);
  rotation_at(m, tau, R);
  position_at(m, tau, pos);
  return world_tri(R, pos, L);
}

template <int kStride>
__device__ __forceinline__ double row_distance(const Staged<kStride>& st, const double* tris, const BodyInfo& A,
                                               const BodyInfo& B, int la, int ia, int lb, int ib,
                                               double tau) {
  stage_pair(st, world_at(A.m, rec(tris, A, la, ia), tau), world_at(B.m, rec(tris, B, lb, ib), tau));
  return __dsqrt_rn(staged_dist_sq(st));
}

// Same row with the lite stage (24 doubles per thread).
template <int kStride>
__device__ __forceinline__ double row_distance_lite(const Staged<kStride>& st, const double* tris,
                                                    const BodyInfo& A, const BodyInfo& B, int la, int ia,
                                                    int lb, int ib, double tau) {
  stage_pair_lite(st, world_at(A.m, rec(tris, A, la, ia), tau), world_at(B.m, rec(tris, B, lb, ib), tau));
  return __dsqrt_rn(staged_dist_sq_lite(st));
}

// ---------------------------------------------------------------- screen

// Per-candidate data the lanes evaluating its rows need (shared memory):
// everything a row needs is one shared-memory read away, no dependent
// global loads (pair -> body -> level table -> record).
struct CandInfo {
  double w0, dt, h, thr, cull_lo, cull_hi;
  int64_t off_a, off_b;  // record indices of the two triangles (tris + off * kRecord)
  int32_t ba, bb, count, first, culled;
  int32_t tab;  // bit 0 / bit 1: the pose table covers side a / b (w0 == 0 and the body's table dt == dt)
};

struct ChildInfo {
  double w0;
  int32_t first, count, pair, ia0, ib0, nb, la, lb;
};

struct ScreenOut {
  Cand* next;
  unsigned long long next_cap;
  const unsigned long long* n_in;  // frontier size on the device (async mode) or null
  unsigned long long* n_out;       // next-frontier counter
  RestRec* resting;
  unsigned long long rest_cap;
  Entry* entries;
  unsigned long long entry_cap;
  Cross* cross;
  unsigned long long cross_cap;
  Counters* ctr;
};

#ifndef LTSG_SCREEN_WARPS
#define LTSG_SCREEN_WARPS 8
#endif
constexpr int kScreenWarps = LTSG_SCREEN_WARPS;
#ifndef LTSG_SCREEN_MINB
#define LTSG_SCREEN_MINB 2
#endif
constexpr int kRowsPerWarp = 32 * kMaxSamples;

__device__ __forceinline__ int sample_count(double span, double speed, double h) {
  // ccd.py:347-352
  if (span == 0.0) return 1;
  if (speed == 0.0) return kMinSamples;
  const double q = ceil(dv(mul(span, speed), mul(0.5, h)));
  long long need;
  if (!(q < 9.2233720368547758e18))  // numpy astype(int) of nan / out of range -> INT64_MIN
    need = (long long)0x8000000000000000ULL;
  else
    need = (long long)q;
  need += 1;
  if (need < kMinSamples) need = kMinSamples;
  if (need > kMaxSamples) need = kMaxSamples;
  return (int)need;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// ---------------------------------------------------------------- poses
// Per-body table of the rigid pose at every sample of the grids
// linspace(0, dt, n), n = 1..33 (561 entries of R row-major + position), for
// the dt of the body's problem: most moving rows start their window at
// w0 = 0 (children inherit w0 = 0 unless an earlier sample flagged), so
// they read their pose instead of recomputing sin/cos and the Rodrigues
// product.  The entries are computed by rotation_at/position_at themselves,
// so a row gets the same bits either way.
constexpr int kPoseEntries = kMaxSamples * (kMaxSamples + 1) / 2;  // 561
constexpr int kPose = 12;

struct PoseTable {
  const double* tab;   // n_bodies x kPoseEntries x kPose, or null
  const double* tdt;   // per body: the dt its table was built for (NaN: none)
  const double* cm;    // n_bodies x kCullM: cull-path motion constants (k_cull_prep), or null
};

// Cull-path motion constants per body: the Rodrigues rotation regrouped as
// R(tau) = base + sin(w tau) (K base) + (1 - cos(w tau)) (K^2 base), for
// cull samples off the pose-table grid (cull arithmetic: FMA allowed, the
// certified margins cover the rounding).
// Layout: [0..2] x0, [3..5] v, [6..14] base, [15..23] K base, [24..32] K^2 base,
// [33] omega, [34] spinning (0/1), [35] pad.
constexpr int kCullM = 36;

__device__ __forceinline__ int grid_entry(int n, int i) { return n * (n - 1) / 2 + i; }

__global__ void k_pose_dt(const PairInfo* __restrict__ pairs, int64_t n_pairs, double* tdt) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_pairs) return;
  const PairInfo p = pairs[k];
  tdt[p.ba] = p.dt;  // a body shared by problems of different dt keeps one of them
  tdt[p.bb] = p.dt;
}

__global__ void k_pose_fill(const BodyInfo* __restrict__ bodies, int n_bodies, const double* __restrict__ tdt,
                            double* __restrict__ tab) {
  const int64_t total = (int64_t)n_bodies * kPoseEntries;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(x / kPoseEntries);
    const int e = (int)(x - (int64_t)b * kPoseEntries);
    int n = 1;
    while (grid_entry(n + 1, 0) <= e) ++n;
    const int i = e - grid_entry(n, 0);
    const double dt = tdt[b];
    if (dt != dt) continue;
    const double tau = linspace_at(0.0, dt, n, i);
    double R[9], pos[3];
    rotation_at(bodies[b].m, tau, R);
    position_at(bodies[b].m, tau, pos);
    double* o = tab + x * kPose;
#pragma unroll
    for (int k = 0; k < 9; ++k) o[k] = R[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) o[9 + k] = pos[k];
  }
}

__global__ void k_cull_prep(const BodyInfo* __restrict__ bodies, int n, double* __restrict__ cm) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const Motion& m = bodies[b].m;
  double* o = cm + (size_t)b * kCullM;
  for (int k = 0; k < 3; ++k) {
    o[k] = m.x0[k];
    o[3 + k] = m.v[k];
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      o[6 + 3 * r + c] = m.base[3 * r + c];
      o[15 + 3 * r + c] = fma(m.K[3 * r + 2], m.base[6 + c], fma(m.K[3 * r + 1], m.base[3 + c], m.K[3 * r] * m.base[c]));
      o[24 + 3 * r + c] = fma(m.KK[3 * r + 2], m.base[6 + c], fma(m.KK[3 * r + 1], m.base[3 + c], m.KK[3 * r] * m.base[c]));
    }
  o[33] = m.omega;
  o[34] = m.spinning ? 1.0 : 0.0;
  o[35] = 0.0;
}

// Pose of body slot `b` at sample i of linspace(w0, dt, n) (= tau).
__device__ __forceinline__ void pose_at(const BodyInfo& B, int b, double tau, bool use_tab, int n, int i,
                                        const PoseTable& pt, double R[9], double pos[3]) {
  if (use_tab) {
    const double2* e = reinterpret_cast<const double2*>(pt.tab + ((size_t)b * kPoseEntries + grid_entry(n, i)) * kPose);
    double v[12];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double2 t = __ldg(e + k);
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = v[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) pos[k] = v[9 + k];
  } else {
    rotation_at(B.m, tau, R);
    position_at(B.m, tau, pos);
  }
}

// Bounding-sphere gap (centre distance minus radii, approximate arithmetic;
// the cull margins cover it) of the candidate's two triangles at sample i.
__device__ __forceinline__ double sphere_gap_at(const BodyInfo* bodies, int ba, int bb, const double* ra,
                                                const double* rb, double tau, int tab, int n, int i,
                                                const PoseTable& pt, double* scale) {
  double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int b = side ? bb : ba;
    const double* r = side ? rb : ra;
    double R[9], pos[3];
    pose_at(bodies[b], b, tau, (tab >> side) & 1, n, i, pt, R, pos);
    const double x = __ldg(r + 12), y = __ldg(r + 13), z = __ldg(r + 14);
    const double cx = fma(R[0], x, fma(R[1], y, fma(R[2], z, pos[0])));  // cull arithmetic: FMA is fine
    const double cy = fma(R[3], x, fma(R[4], y, fma(R[5], z, pos[1])));
    const double cz = fma(R[6], x, fma(R[7], y, fma(R[8], z, pos[2])));
    if (side) { bx = cx; by = cy; bz = cz; } else { ax = cx; ay = cy; az = cz; }
  }
  const double dx = ax - bx, dy = ay - by, dz = az - bz;
  const double rA = __ldg(ra + 15), rB = __ldg(rb + 15);
  *scale = 1.0 + fabs(ax) + fabs(ay) + fabs(az) + fabs(bx) + fabs(by) + fabs(bz) + rA + rB;
  return sqrt(fma(dx, dx, fma(dy, dy, dz * dz))) - (rA + rB);
}

// Exact 15-feature distance of one row, triangles posed at sample i.
template <int kStride>
__device__ __forceinline__ double row_distance_posed(const Staged<kStride>& st, const BodyInfo* bodies, int ba,
                                                     int bb, const double* ra, const double* rb, double tau,
                                                     int tab, int n, int i, const PoseTable& pt) {
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int b = side ? bb : ba;
    const BodyInfo& B = bodies[b];
    double R[9], pos[3], L[9];
    pose_at(B, b, tau, (tab >> side) & 1, n, i, pt, R, pos);
    load_local(side ? rb : ra, L);
    const Tri t = world_tri(R, pos, L);
    const int base = side ? kLiteB : kLiteA;
#pragma unroll
    for (int k = 0; k < 3; ++k) st.put(base + 3 * k, t.v[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const V3 e = t.v[(k + 1) % 3] - t.v[k];
      st.at((side ? kLiteBB : kLiteAA) + k) = dot_simd(e, e);
    }
  }
  return __dsqrt_rn(staged_dist_sq_lite(st));
}

// Separating-axis cull of one moving row (same certificate as sat_cull on
// static records): world corners at the row's pose (FMA arithmetic -- cull
// data, not reference arithmetic), axes = both face normals and the
// centroid direction, compared without normalising (gap > T |u|).
__device__ __forceinline__ void world_corners_fast(const double R[9], const double pos[3], const double* r,
                                                   double w[9]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = __ldg(r + 3 * k), y = __ldg(r + 3 * k + 1), z = __ldg(r + 3 * k + 2);
    w[3 * k] = fma(R[0], x, fma(R[1], y, fma(R[2], z, pos[0])));
    w[3 * k + 1] = fma(R[3], x, fma(R[4], y, fma(R[5], z, pos[1])));
    w[3 * k + 2] = fma(R[6], x, fma(R[7], y, fma(R[8], z, pos[2])));
  }
}

__device__ __forceinline__ double axis_gap(double ux, double uy, double uz, const double a[9], const double b[9]) {
  double alo = 0.0, ahi = 0.0, blo = 0.0, bhi = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = fma(ux, a[3 * k], fma(uy, a[3 * k + 1], uz * a[3 * k + 2]));
    const double y = fma(ux, b[3 * k], fma(uy, b[3 * k + 1], uz * b[3 * k + 2]));
    alo = k ? fmin(alo, x) : x;
    ahi = k ? fmax(ahi, x) : x;
    blo = k ? fmin(blo, y) : y;
    bhi = k ? fmax(bhi, y) : y;
  }
  return fmax(blo - ahi, alo - bhi);
}

__device__ __forceinline__ bool sat_cull_posed(const BodyInfo* bodies, int ba, int bb, const double* ra,
                                               const double* rb, double tau, int tab, int n, int i,
                                               const PoseTable& pt, double thr) {
  if (__ldg(ra + 15) < 0.0 || __ldg(rb + 15) < 0.0) return false;  // slivers are never culled
  double a[9], b[9];
  {
    double R[9], pos[3];
    pose_at(bodies[ba], ba, tau, tab & 1, n, i, pt, R, pos);
    world_corners_fast(R, pos, ra, a);
    pose_at(bodies[bb], bb, tau, (tab >> 1) & 1, n, i, pt, R, pos);
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

// Screen one frontier (one generation): every candidate is sampled over
// [w0, dt] (ccd.py:321-370) and decided (ccd.py:404-446).  A warp owns 32
// consecutive candidates; their 1..33 samples are flattened into rows and
// spread over the 32 lanes, so lanes stay busy whatever the sample counts.
__global__ void __launch_bounds__(32 * kScreenWarps, LTSG_SCREEN_MINB)
k_screen(const Cand* __restrict__ front, int64_t n, const PairInfo* __restrict__ pairs,
         const BodyInfo* __restrict__ bodies, const double* __restrict__ tris, ScreenOut out, PoseTable pt) {
  if (out.n_in) n = (int64_t)min(*out.n_in, out.next_cap);
  __shared__ union {  // per warp: candidate info, later reused for child descriptors
    CandInfo cand[32];
    ChildInfo child[32];
  } s_u[kScreenWarps];
  __shared__ uint8_t s_bits[kScreenWarps][kRowsPerWarp];
  __shared__ int16_t s_queue[kScreenWarps][kRowsPerWarp];
  extern __shared__ double s_stage[];  // kStagedLite x (32 * kScreenWarps), dynamic
  const Staged<32 * kScreenWarps> st{s_stage + threadIdx.x};
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (n + 31) / 32;
  CandInfo* info = s_u[warp].cand;
  ChildInfo* kid = s_u[warp].child;
  uint8_t* bits = s_bits[warp];
  int16_t* queue = s_queue[warp];
  unsigned long long acc_rows = 0, acc_exact = 0, acc_window = 0, acc_sphere = 0;

  for (int64_t wi = blockIdx.x * (int64_t)kScreenWarps + warp; wi < n_warps;
       wi += (int64_t)gridDim.x * kScreenWarps) {
    const int64_t ci = wi * 32 + lane;
    const bool valid = ci < n;
    CandInfo me{};
    Cand own{};        // the candidate itself (this lane's, for the decisions)
    double speed = 0;  // its Lipschitz speed (entries carry it)
    if (valid) {
      const Cand c = front[ci];
      own = c;
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
      speed = sp;
      me.w0 = c.w0;
      me.tab = (pt.tab != nullptr && c.w0 == 0.0)
          ? ((pt.tdt[p.ba] == p.dt ? 1 : 0) | (pt.tdt[p.bb] == p.dt ? 2 : 0)) : 0;
      me.dt = p.dt;
      const double span = fmax(sub(p.dt, c.w0), 0.0);
      me.count = sample_count(span, sp, me.h);
      const double step = me.count > 1
          ? sub(linspace_at(c.w0, p.dt, me.count, 1), linspace_at(c.w0, p.dt, me.count, 0)) : 0.0;
      me.thr = add(me.h, mul(mul(0.5, sp), step));  // ccd.py:410-411
      // Certified cull window.  The bounding-sphere gap g(tau) of the pair is
      // `speed`-Lipschitz (every point of a triangle moves at most
      // |v| + omega*arm, the reference's own bound, ccd.py:340-345), and the
      // true triangle distance is >= g.  With g evaluated at both window
      // ends, samples before t_lo or after t_hi provably clear every
      // threshold (flag, touch, rest) of this candidate.
      me.cull_lo = -1.0;
      me.cull_hi = 2.0 * p.dt + 1.0;
      if (__ldg(ra_ + 15) >= 0.0 && __ldg(rb_ + 15) >= 0.0) {
        const double T = fmax(me.thr, add(me.h, kRestSlop));
        double sc0 = 0.0, sc1 = 0.0;
        // (the gap call sets the scale: evaluate it before reading sc0/sc1)
        const double gap0 = sphere_gap_at(bodies, p.ba, p.bb, ra_, rb_, c.w0, me.tab, me.count, 0, pt, &sc0);
        const double g0 = gap0 - (T + kCullMargin * sc0);
        double g1 = g0;
        if (p.dt > c.w0) {
          const double gap1 = sphere_gap_at(bodies, p.ba, p.bb, ra_, rb_, p.dt, me.tab, me.count, me.count - 1, pt,
                                            &sc1);
          g1 = gap1 - (T + kCullMargin * sc1);
        }
        if (sp > 0.0) {
          me.cull_lo = c.w0 + g0 / sp;  // rows with tau < cull_lo are cleared
          me.cull_hi = p.dt - g1 / sp;  // rows with tau > cull_hi are cleared
        } else if (g0 > 0.0) {
          me.cull_lo = 2.0 * p.dt + 1.0;  // no motion: the whole window clears
        }
        // every sample cleared?
        me.culled = me.cull_lo > p.dt || me.cull_hi < c.w0 || me.cull_lo > me.cull_hi;
      }
    }
    // rows of culled candidates are decided (all flags false) without being evaluated
    const int nrows = me.culled ? 0 : me.count;
    const int incl = warp_incl_scan(nrows, lane);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int all_rows = me.count;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) all_rows += __shfl_xor_sync(0xffffffffu, all_rows, o);
    me.first = incl - nrows;
    info[lane] = me;
    __syncwarp();

    // (a) per-row certified sphere cull at the row's own tau: the bounding
    // spheres of both triangles are moved to tau (same rigid motion as the
    // triangles); rows whose gap exceeds every threshold plus the margin
    // are decided (no flag, not below, not resting).  Survivors are queued.
    int nq = 0;
    for (int r0 = 0; r0 < total; r0 += 32) {
      const int r = r0 + lane;
      bool keep = false;
      if (r < total) {
        int o = 0;  // owner: last lane with first <= r among lanes that own rows
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (info[o + step].first <= r) o += step;
        while (info[o].culled || info[o].count == 0) --o;
        const CandInfo& c = info[o];
        const int i = r - c.first;
        const double tau = linspace_at(c.w0, c.dt, c.count, i);
        const double* ra_ = tris + c.off_a * kRecord;
        const double* rb_ = tris + c.off_b * kRecord;
        keep = !(tau < c.cull_lo || tau > c.cull_hi);
        if (keep && __ldg(ra_ + 15) >= 0.0 && __ldg(rb_ + 15) >= 0.0) {
          double scale;
          const double gap = sphere_gap_at(bodies, c.ba, c.bb, ra_, rb_, tau, c.tab, c.count, i, pt, &scale);
          keep = !(gap > fmax(c.thr, add(c.h, kRestSlop)) + kCullMargin * scale);
        }
        if (!keep) bits[r] = 0;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) queue[nq + __popc(m & ((1u << lane) - 1u))] = (int16_t)r;
      nq += __popc(m);
    }
    __syncwarp();
    const int nq_sphere = nq;
    // (b1) separating-axis cull of the sphere survivors, densely; survivors
    // are compacted in place (a chunk is read before any lane writes)
    {
      int nq2 = 0;
      for (int q0 = 0; q0 < nq; q0 += 32) {
        const int q = q0 + lane;
        bool keep = false;
        int r = 0;
        if (q < nq) {
          r = queue[q];
          int o = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1)
            if (info[o + step].first <= r) o += step;
          while (info[o].culled || info[o].count == 0) --o;
          const CandInfo& c = info[o];
          const int i = r - c.first;
          const double tau = linspace_at(c.w0, c.dt, c.count, i);
          keep = !sat_cull_posed(bodies, c.ba, c.bb, tris + c.off_a * kRecord, tris + c.off_b * kRecord, tau, c.tab,
                                 c.count, i, pt, fmax(c.thr, add(c.h, kRestSlop)));
          if (!keep) bits[r] = 0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) queue[nq2 + __popc(m & ((1u << lane) - 1u))] = (int16_t)r;
        nq2 += __popc(m);
      }
      nq = nq2;
    }
    __syncwarp();
    // (b) exact 15-feature distance of the surviving rows, densely
    for (int q = lane; q < nq; q += 32) {
      const int r = queue[q];
      int o = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (info[o + step].first <= r) o += step;
      while (info[o].culled || info[o].count == 0) --o;
      const CandInfo& c = info[o];
      const int i = r - c.first;
      const double tau = linspace_at(c.w0, c.dt, c.count, i);
      const double d = row_distance_posed(st, bodies, c.ba, c.bb, tris + c.off_a * kRecord, tris + c.off_b * kRecord,
                                          tau, c.tab, c.count, i, pt);
      uint8_t b = 0;
      if (d <= c.thr) b |= 1;                  // screen flag
      if (d <= c.h) b |= 2;                    // at or below touching distance
      if (d <= add(c.h, kRestSlop)) b |= 4;    // resting test (ccd.py:407)
      bits[r] = b;
    }
    __syncwarp();

    // per-candidate decisions
    ChildInfo ch{};
    if (valid && !me.culled) {
      const uint8_t* cb = bits + me.first;
      const bool fine = own.la == 0 && own.lb == 0;
      if (fine && me.w0 == 0.0 && (cb[0] & 4)) {
        const unsigned long long slot = atomicAdd(&out.ctr->resting, 1ULL);
        if (slot < out.rest_cap) out.resting[slot] = RestRec{own.pair, own.ia, own.ib, 0, me.h};
      } else {
        int k0 = -1;
        for (int k = 0; k < me.count; ++k)
          if (cb[k] & 1) { k0 = k; break; }
        if (k0 >= 0 && !fine) {  // ccd.py:414-428
          ch.w0 = linspace_at(me.w0, me.dt, me.count, k0 > 0 ? k0 - 1 : 0);
          ch.pair = own.pair;
          int na = 1, nb = 1;
          ch.ia0 = own.ia;
          ch.ib0 = own.ib;
          if (own.la > 0) {
            const int2 cr = *reinterpret_cast<const int2*>(tris + me.off_a * kRecord + 11);
            ch.ia0 = cr.x;
            na = cr.y;
          }
          if (own.lb > 0) {
            const int2 cr = *reinterpret_cast<const int2*>(tris + me.off_b * kRecord + 11);
            ch.ib0 = cr.x;
            nb = cr.y;
          }
          ch.nb = nb;
          ch.count = na * nb;
          ch.la = own.la > 0 ? own.la - 1 : 0;
          ch.lb = own.lb > 0 ? own.lb - 1 : 0;
        } else if (k0 >= 0) {  // fine: flagged runs (ccd.py:429-446)
          int k = k0;
          while (k < me.count) {
            if (!(cb[k] & 1)) { ++k; continue; }
            int ke = k;
            while (ke + 1 < me.count && (cb[ke + 1] & 1)) ++ke;
            const int lo_i = k > 0 ? k - 1 : 0;
            const int hi_i = ke + 1 < me.count - 1 ? ke + 1 : me.count - 1;
            if (cb[lo_i] & 2) {
              const unsigned long long slot = atomicAdd(&out.ctr->cross, 1ULL);
              if (slot < out.cross_cap)
                out.cross[slot] = Cross{own.pair, own.ia, own.ib, 0,
                                        linspace_at(me.w0, me.dt, me.count, lo_i), me.h};
            } else if (hi_i > lo_i) {
              const unsigned long long slot = atomicAdd(&out.ctr->entries, 1ULL);
              if (slot < out.entry_cap)
                out.entries[slot] = Entry{own.pair, own.ia, own.ib, 0,
                                          linspace_at(me.w0, me.dt, me.count, lo_i),
                                          linspace_at(me.w0, me.dt, me.count, hi_i), me.h, speed};
            }
            k = ke + 1;
          }
        }
      }
    }
    // cooperative, coalesced child emission
    const int cincl = warp_incl_scan(ch.count, lane);
    const int ctotal = __shfl_sync(0xffffffffu, cincl, 31);
    unsigned long long cbase = 0;
    acc_rows += (unsigned long long)all_rows;  // warp-uniform; flushed once per warp
    acc_exact += (unsigned long long)nq;
    acc_window += (unsigned long long)total;
    acc_sphere += (unsigned long long)nq_sphere;
    if (lane == 0 && ctotal) cbase = atomicAdd(out.n_out, (unsigned long long)ctotal);
    cbase = __shfl_sync(0xffffffffu, cbase, 0);
    if (ctotal) {
      ch.first = cincl - ch.count;
      __syncwarp();  // cand and child info share storage
      kid[lane] = ch;
      __syncwarp();
      for (int s = lane; s < ctotal; s += 32) {
        int o = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (kid[o + step].first <= s) o += step;
        const ChildInfo& c = kid[o];
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
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (acc_rows) atomicAdd(&out.ctr->rows, acc_rows);
    if (acc_exact) atomicAdd(&out.ctr->screen_exact, acc_exact);
    if (acc_window) atomicAdd(&out.ctr->rows_window, acc_window);
    if (acc_sphere) atomicAdd(&out.ctr->rows_sphere, acc_sphere);
  }
}


#include "moving.cuh"

// ---------------------------------------------------------------- static screen

// World records at tau = 0 (the pose at the window start), 20 doubles each:
//   [0..8]  world corners x = base * local + x0 in the reference's einsum
//           order -- exactly what rotation_at/position_at give at tau = 0
//   [9] epsilon, [10] arm, [11] children (copied from the body record)
//   [12..14] bounding-sphere centre (corner mean), [15] radius, or -1 when
//           the triangle is a sliver (cond = Lmax^2 / |e0 x e2| > 1e4)
//   [16..18] unit face normal n, [19] plane offset n . v0 (cull data only)

__global__ void k_world_count(const BodyInfo* __restrict__ bodies, int n, int64_t* cnt) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > n) return;
  if (b == n) {
    cnt[n] = 0;
    return;
  }
  const BodyInfo& B = bodies[b];
  const int top = B.n_levels - 1;
  cnt[b] = B.level_off[top] + B.level_size[top] - B.level_off[0];
}

#ifndef LTSG_WORLD_MINB
#define LTSG_WORLD_MINB 8
#endif
#ifndef LTSG_WORLD_STAGE
#define LTSG_WORLD_STAGE 1
#endif
__global__ void __launch_bounds__(128, LTSG_WORLD_MINB) k_world_fill(const BodyInfo* __restrict__ bodies, int n,
                                                    const int64_t* __restrict__ woff,
                                                    const double* __restrict__ tris, double* __restrict__ world,
                                                    double* __restrict__ wsph) {
  // One world record per lane, warps independent (no block barriers): the
  // 8 record loads of a lane are all in flight at once.  A warp covers 32
  // consecutive world records; their bodies are found by one binary search
  // (lane 0) and a short forward walk per lane.
  const int lane = threadIdx.x & 31;
  const int64_t n_world = woff[n];
#if LTSG_WORLD_STAGE
  __shared__ double2 s_stage_w[4][32 * (kWorld / 2)];  // 128 threads = 4 warps
  double2* stage = s_stage_w[threadIdx.x >> 5];
#endif
  for (int64_t w0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < n_world;
       w0 += (int64_t)gridDim.x * blockDim.x) {
    int b0 = 0;
    if (lane == 0) {
      int lo = 0, hi = n;  // last b with woff[b] <= w0
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(woff + mid) <= w0) lo = mid; else hi = mid;
      }
      b0 = lo;
    }
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    const int64_t w = w0 + lane;
    const bool valid = w < n_world;
    if (valid) {
      int b = b0;
      while (__ldg(woff + b + 1) <= w) ++b;
      const int64_t j = w - woff[b];
      const BodyInfo& B = bodies[b];
      const double2* src = reinterpret_cast<const double2*>(tris + (size_t)(B.level_off[0] + j) * kRecord);
      double r[kRecord];
#pragma unroll
      for (int k = 0; k < kRecord / 2; ++k) {
        const double2 v = __ldg(src + k);
        r[2 * k] = v.x;
        r[2 * k + 1] = v.y;
      }
      double pos[3];
      position_at(B.m, 0.0, pos);
      const Tri t = world_tri(B.m.base, pos, r);
      double wr[kWorld];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        wr[3 * k] = t.v[k].x;
        wr[3 * k + 1] = t.v[k].y;
        wr[3 * k + 2] = t.v[k].z;
      }
      wr[9] = r[9];
      wr[10] = r[10];
      {  // first child as an absolute world index (children are contiguous)
        int lvl = 0;
        while (lvl + 1 < B.n_levels && B.level_off[0] + j >= B.level_off[lvl + 1]) ++lvl;
        int2 ch = *reinterpret_cast<const int2*>(r + 11);
        if (lvl > 0) ch.x = (int32_t)(woff[b] + B.level_off[lvl - 1] - B.level_off[0] + ch.x);
        *reinterpret_cast<int2*>(wr + 11) = ch;
      }
      // bounding sphere in world coordinates (approximate; the cull margin absorbs it)
      constexpr double kThird = 1.0 / 3.0;
      const V3 c{(t.v[0].x + t.v[1].x + t.v[2].x) * kThird, (t.v[0].y + t.v[1].y + t.v[2].y) * kThird,
                 (t.v[0].z + t.v[1].z + t.v[2].z) * kThird};
      double r2 = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const V3 d = t.v[k] - c;
        r2 = fmax(r2, fma(d.x, d.x, fma(d.y, d.y, d.z * d.z)));
      }
      // unit face normal and plane offset for the separating-axis cull
      const V3 e1{t.v[1].x - t.v[0].x, t.v[1].y - t.v[0].y, t.v[1].z - t.v[0].z};
      const V3 e2{t.v[2].x - t.v[0].x, t.v[2].y - t.v[0].y, t.v[2].z - t.v[0].z};
      const V3 nn{fma(e1.y, e2.z, -e1.z * e2.y), fma(e1.z, e2.x, -e1.x * e2.z), fma(e1.x, e2.y, -e1.y * e2.x)};
      const double nl = sqrt(fma(nn.x, nn.x, fma(nn.y, nn.y, nn.z * nn.z)));
      const double inv = nl > 0.0 ? 1.0 / nl : 0.0;
      wr[16] = nn.x * inv;
      wr[17] = nn.y * inv;
      wr[18] = nn.z * inv;
      wr[19] = fma(wr[16], t.v[0].x, fma(wr[17], t.v[0].y, wr[18] * t.v[0].z));
      wr[12] = c.x;
      wr[13] = c.y;
      wr[14] = c.z;
      // sliver flag from the body record; a zero-area triangle is never culled either
      wr[15] = r[15] >= 0.0 && nl > 0.0 ? sqrt(r2) * (1.0 + 1e-12) : -1.0;
#if LTSG_WORLD_STAGE
#pragma unroll
      for (int k = 0; k < kWorld / 2; ++k) stage[lane * (kWorld / 2) + k] = make_double2(wr[2 * k], wr[2 * k + 1]);
#else
      double2* dst = reinterpret_cast<double2*>(world + (size_t)w * kWorld);
#pragma unroll
      for (int k = 0; k < kWorld / 2; ++k) dst[k] = make_double2(wr[2 * k], wr[2 * k + 1]);
#endif
      double2* sp = reinterpret_cast<double2*>(wsph + (size_t)w * kSph);
      sp[0] = make_double2(c.x, c.y);
      sp[1] = make_double2(c.z, wr[15] < 0.0 ? -1.0 : wr[15] + r[9]);
    }
#if LTSG_WORLD_STAGE
    // the warp's records are consecutive in `world`: write them out from the
    // stage with contiguous 16-byte stores
    __syncwarp();
    const int nv = (int)min((int64_t)32, n_world - w0);
    double2* dst = reinterpret_cast<double2*>(world + (size_t)w0 * kWorld);
    for (int idx = lane; idx < nv * (kWorld / 2); idx += 32) dst[idx] = stage[idx];
    __syncwarp();
#endif
  }
}

__device__ __forceinline__ Tri load_world(const double* w) {
  const double2* q = reinterpret_cast<const double2*>(w);
  Tri t;
  double v[10];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double2 x = __ldg(q + k);
    v[2 * k] = x.x;
    v[2 * k + 1] = x.y;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) t.v[k] = V3{v[3 * k], v[3 * k + 1], v[3 * k + 2]};
  return t;
}

// Certified "cannot touch": the bounding spheres are farther apart than
// thr plus a margin.  Every witness point the reference computes lies on
// its triangle up to rounding (segment parameters are clipped to [0,1];
// point-triangle weights are in [0,1]; face points of non-sliver triangles
// stay within rounding of the face), so its 15-feature distance is at least
// the true triangle distance minus rounding, and the true distance is at
// least the sphere gap.  Slivers (radius slot < 0) are never culled.
__device__ __forceinline__ bool sphere_cull(const double* wa, const double* wb, double thr) {
  const double ra = __ldg(wa + 15), rb = __ldg(wb + 15);
  if (ra < 0.0 || rb < 0.0) return false;
  const double dx = __ldg(wa + 12) - __ldg(wb + 12);
  const double dy = __ldg(wa + 13) - __ldg(wb + 13);
  const double dz = __ldg(wa + 14) - __ldg(wb + 14);
  const double scale = 1.0 + fabs(__ldg(wa + 12)) + fabs(__ldg(wa + 13)) + fabs(__ldg(wa + 14)) + ra + rb;
  const double reach = ra + rb + thr + kCullMargin * scale;
  return dx * dx + dy * dy + dz * dz > reach * reach;
}

// Certified separating-axis cull on static world records.  For any direction
// u the gap between the projections of the two triangles onto u, divided by
// |u|, is a lower bound of their distance; the axes are both face normals
// (a triangle projects onto its own normal as the single value n . v0) and
// the centroid direction.  The same rounding argument as sphere_cull applies
// (the margin is far above the few-ulp error of these dot products), and
// slivers or zero-area triangles (radius slot < 0) are never culled.  This is
// cull arithmetic, not reference arithmetic: it may use FMA freely.
__device__ __forceinline__ bool sat_cull(const double* wa, const double* wb, double thr) {
  const double ra = __ldg(wa + 15), rb = __ldg(wb + 15);
  if (ra < 0.0 || rb < 0.0) return false;
  // loads are staged axis by axis (corners re-read from L1) to keep the
  // register footprint low: the filter kernel runs at high occupancy
  const double ca0 = __ldg(wa + 12), ca1 = __ldg(wa + 13), ca2 = __ldg(wa + 14);
  const double cb0 = __ldg(wb + 12), cb1 = __ldg(wb + 13), cb2 = __ldg(wb + 14);
  const double scale = 1.0 + fabs(ca0) + fabs(ca1) + fabs(ca2) + fabs(cb0) + fabs(cb1) + fabs(cb2) + ra + rb;
  const double T = thr + kCullMargin * scale;
  // a face normal against the other triangle's corners (the own triangle
  // projects to the single value n . v0 stored in slot 19)
  auto face_gap = [&](const double* w, const double* o) {
    const double2 n01 = __ldg(reinterpret_cast<const double2*>(w + 16));
    const double2 n2d = __ldg(reinterpret_cast<const double2*>(w + 18));
    double lo = 0.0, hi = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double x = fma(n01.x, __ldg(o + 3 * k), fma(n01.y, __ldg(o + 3 * k + 1), n2d.x * __ldg(o + 3 * k + 2)));
      lo = k ? fmin(lo, x) : x;
      hi = k ? fmax(hi, x) : x;
    }
    return fmax(lo - n2d.y, n2d.y - hi);
  };
  if (face_gap(wa, wb) > T) return true;
  if (face_gap(wb, wa) > T) return true;
  // centroid direction
  const double u0 = cb0 - ca0, u1 = cb1 - ca1, u2 = cb2 - ca2;
  const double len = sqrt(fma(u0, u0, fma(u1, u1, u2 * u2)));
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

constexpr int kStaticWarps = 4;
#ifndef LTSG_STATIC_LITE
#define LTSG_STATIC_LITE 1
#endif
constexpr int kStaticStageBytes = (LTSG_STATIC_LITE ? kStagedLite : kStaged) * 32 * kStaticWarps * sizeof(double);
#ifndef LTSG_STATIC_MINB
#define LTSG_STATIC_MINB 7
#endif
#ifndef LTSG_STATIC_GRID
#define LTSG_STATIC_GRID 20
#endif

// Static batches (every problem has dt = 0) run a leaner traversal.  Every
// candidate has exactly one sample at tau = w0 = 0 (span 0, ccd.py:352), its
// flag threshold is h (step 0, ccd.py:410-411) and a fine candidate within
// h + 1e-9 is resting (ccd.py:407-409).  Candidates carry absolute indices
// of their world records (Cand::ia/ib), and a child is tested against the
// certified sphere cull the moment it is emitted: a culled child is a
// decided row (not flagged, not resting) and is only counted, so the next
// frontier holds exactly the rows that need the 15-feature distance.
// Compact cull spheres of the world records, one 32-B sector each:
// (centre, R = radius + epsilon), R = -1 for slivers.  The sphere test of a
// child pair reads two sectors instead of four, and the whole array of a
// c1 batch (112 MB) stays L2-resident.
__device__ __forceinline__ bool static_child_cull(const double* __restrict__ wsph, int32_t wa, int32_t wb) {
  const double2* pa = reinterpret_cast<const double2*>(wsph + (size_t)wa * kSph);
  const double2* pb = reinterpret_cast<const double2*>(wsph + (size_t)wb * kSph);
  const double2 a01 = __ldg(pa), a2r = __ldg(pa + 1), b01 = __ldg(pb), b2r = __ldg(pb + 1);
  if (a2r.y < 0.0 || b2r.y < 0.0) return false;  // slivers are never culled
  const double dx = a01.x - b01.x, dy = a01.y - b01.y, dz = a2r.x - b2r.x;
  // same certificate as sphere_cull with thr = eps_a + eps_b + 1e-9 folded into R
  const double scale = 1.0 + fabs(a01.x) + fabs(a01.y) + fabs(a2r.x) + a2r.y + b2r.y;
  const double reach = a2r.y + b2r.y + kRestSlop + kCullMargin * scale;
  return fma(dx, dx, fma(dy, dy, dz * dz)) > reach * reach;
}

// Seeds (roots x roots per pair, ccd.py:385-391) in world indices, culled
// (sphere, then separating axes): the frontier holds only exact rows.
__global__ void k_seed_static(const PairInfo* __restrict__ pairs, int64_t n_pairs,
                              const BodyInfo* __restrict__ bodies, const int64_t* __restrict__ woff,
                              const double* __restrict__ world, const double* __restrict__ wsph, Cand* out,
                              unsigned long long cap, Counters* ctr, unsigned long long* n_out, int exhaustive) {
  const int lane = threadIdx.x & 31;
  unsigned long long culled = 0;
  for (int64_t k = blockIdx.x; k < n_pairs; k += gridDim.x) {
    const PairInfo p = pairs[k];
    const BodyInfo& A = bodies[p.ba];
    const BodyInfo& B = bodies[p.bb];
    const int la = exhaustive ? 0 : A.n_levels - 1, lb = exhaustive ? 0 : B.n_levels - 1;
    const int64_t na = A.level_size[la], nb = B.level_size[lb];
    const int64_t a0 = woff[p.ba] + A.level_off[la] - A.level_off[0];
    const int64_t b0 = woff[p.bb] + B.level_off[lb] - B.level_off[0];
    for (int64_t j0 = threadIdx.x - lane; j0 < na * nb; j0 += blockDim.x) {
      const int64_t j = j0 + lane;
      bool keep = false;
      int32_t wa = 0, wb = 0;
      if (j < na * nb) {
        wa = (int32_t)(a0 + j / nb);
        wb = (int32_t)(b0 + j % nb);
        keep = !static_child_cull(wsph, wa, wb);
        if (keep) {
          const double* pa = world + (size_t)wa * kWorld;
          const double* pb = world + (size_t)wb * kWorld;
          keep = !sat_cull(pa, pb, add(add(__ldg(pa + 9), __ldg(pb + 9)), kRestSlop));
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int nvalid = (int)min((int64_t)32, na * nb - j0);
      culled += (unsigned long long)nvalid;  // every seed is a test; survivors go to the exact pass
      unsigned long long base = 0;
      if (lane == 0 && m) base = atomicAdd(n_out, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const unsigned long long dst = base + __popc(m & ((1u << lane) - 1u));
        if (dst < cap) out[dst] = Cand{(int32_t)k, wa, wb, (int16_t)la, (int16_t)lb, 0.0};
      }
    }
  }
  if (lane == 0 && culled) atomicAdd(&ctr->rows, culled);
}

// Exhaustive static seeds (fine x fine rows of every pair, ccd.py:385-391)
// as sphere-test tiles: a work item is (pair, 128 triangles of a, 32 of b);
// the b tile's compact spheres are staged in shared memory and read by every
// lane at the same address, each lane holds its a sphere in registers, so a
// row's certified sphere test (static_child_cull's certificate) is a dozen
// FP64 operations on registers.  Survivors take the separating-axis cull and
// are appended to the exact frontier.  Every row is counted as a test.
constexpr int kSeedTileA = 128, kSeedTileB = 32;

__global__ void k_seed_tile_count(const PairInfo* pairs, int64_t n, const BodyInfo* bodies, int64_t* count) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k > n) return;
  if (k == n) {
    count[n] = 0;
    return;
  }
  int la, lb;
  int64_t na, nb;
  seed_levels(pairs[k], bodies, 1, &la, &lb, &na, &nb);
  count[k] = ((na + kSeedTileA - 1) / kSeedTileA) * ((nb + kSeedTileB - 1) / kSeedTileB);
}

__global__ void __launch_bounds__(kSeedTileA)
k_seed_static_tile(const PairInfo* __restrict__ pairs, int64_t n_pairs, const BodyInfo* __restrict__ bodies,
                   const int64_t* __restrict__ woff, const double* __restrict__ world,
                   const double* __restrict__ wsph, const int64_t* __restrict__ item_off, Cand* out,
                   unsigned long long cap, Counters* ctr, unsigned long long* n_out) {
  __shared__ double4 sB[kSeedTileB];
  const int lane = threadIdx.x & 31;
  const int64_t n_items = item_off[n_pairs];
  unsigned long long rows = 0;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    int64_t lo = 0, hi = n_pairs;  // last pair with item_off[k] <= item
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(item_off + mid) <= item) lo = mid; else hi = mid;
    }
    const PairInfo p = pairs[lo];
    int la, lb;
    int64_t na, nb;
    seed_levels(p, bodies, 1, &la, &lb, &na, &nb);
    const int64_t tiles_b = (nb + kSeedTileB - 1) / kSeedTileB;
    const int64_t local = item - item_off[lo];
    const int64_t ta = local / tiles_b, tb = local - ta * tiles_b;
    const int64_t a0 = woff[p.ba] + ta * kSeedTileA, b0 = woff[p.bb] + tb * kSeedTileB;
    const int nat = (int)min((int64_t)kSeedTileA, na - ta * kSeedTileA);
    const int nbt = (int)min((int64_t)kSeedTileB, nb - tb * kSeedTileB);
    __syncthreads();
    if (threadIdx.x < nbt) {
      const double2* q = reinterpret_cast<const double2*>(wsph + (size_t)(b0 + threadIdx.x) * kSph);
      const double2 x = __ldg(q), y = __ldg(q + 1);
      sB[threadIdx.x] = make_double4(x.x, x.y, y.x, y.y);
    }
    __syncthreads();
    if (threadIdx.x == 0) rows += (unsigned long long)nat * (unsigned long long)nbt;
    const bool valid = threadIdx.x < nat;
    const int32_t wa = (int32_t)(a0 + (valid ? threadIdx.x : 0));
    const double2* qa = reinterpret_cast<const double2*>(wsph + (size_t)wa * kSph);
    const double2 a01 = __ldg(qa), a2r = __ldg(qa + 1);
    const double base = 1.0 + fabs(a01.x) + fabs(a01.y) + fabs(a2r.x) + a2r.y;
    // the sphere tests of 4 rows per step (independent chains); the rare
    // survivors take the separating-axis cull in place
#pragma unroll 4
    for (int j = 0; j < nbt; ++j) {
      const double4 b = sB[j];
      bool keep = false;
      if (valid) {
        if (a2r.y < 0.0 || b.w < 0.0) {
          keep = true;  // slivers are never culled
        } else {  // static_child_cull's certificate, same arithmetic
          const double dx = a01.x - b.x, dy = a01.y - b.y, dz = a2r.x - b.z;
          const double reach = a2r.y + b.w + kRestSlop + kCullMargin * (base + b.w);
          keep = !(fma(dx, dx, fma(dy, dy, dz * dz)) > reach * reach);
        }
      }
      if (__any_sync(0xffffffffu, keep)) {
        if (keep) {
          const int32_t wb = (int32_t)(b0 + j);
          const double* pa = world + (size_t)wa * kWorld;
          const double* pb = world + (size_t)wb * kWorld;
          keep = !sat_cull(pa, pb, add(add(__ldg(pa + 9), __ldg(pb + 9)), kRestSlop));
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (m) {
          unsigned long long slot = 0;
          if (lane == 0) slot = atomicAdd(n_out, (unsigned long long)__popc(m));
          slot = __shfl_sync(0xffffffffu, slot, 0);
          if (keep) {
            const unsigned long long dst = slot + __popc(m & ((1u << lane) - 1u));
            if (dst < cap) out[dst] = Cand{(int32_t)lo, wa, (int32_t)(b0 + j), 0, 0, 0.0};
          }
        }
      }
    }
  }
  if (threadIdx.x == 0 && rows) atomicAdd(&ctr->rows, rows);
}

// A flagged coarse row of a static generation: its na x nb children
// (ccd.py:418-427) in absolute world indices.
struct Parent {
  int32_t pair, a0, b0;
  uint8_t na, nb, la, lb;
};
static_assert(sizeof(Parent) == 16, "Parent layout");
static_assert(sizeof(Parent) <= sizeof(Cand), "parents are stored in a candidate buffer");

// The decision of a static row known to be at or below its threshold
// (`hit`): a resting record for a fine row (ccd.py:407-409), a Parent for a
// flagged coarse row (ccd.py:410-411), appended with one atomic per warp.
// Warp-uniform call (every lane of the warp calls it; `hit` false for idle lanes).
__device__ __forceinline__ void static_row_hit(bool hit, int64_t ci, const Cand* __restrict__ front,
                                               const PairInfo* __restrict__ pairs, const double* __restrict__ world,
                                               const int64_t* __restrict__ woff, const ScreenOut& out,
                                               Parent* __restrict__ par, unsigned long long* n_par, int lane) {
  bool flagged = false, rest = false;
  Parent P{};
  RestRec R{};
  if (hit) {
    const Cand c = front[ci];
    const double* wa = world + (size_t)c.ia * kWorld;
    const double* wb = world + (size_t)c.ib * kWorld;
    if (c.la == 0 && c.lb == 0) {
      const PairInfo p = pairs[c.pair];
      const double h = add(__ldg(wa + 9), __ldg(wb + 9));
      R = RestRec{c.pair, (int32_t)(c.ia - woff[p.ba]), (int32_t)(c.ib - woff[p.bb]), 0, h};
      rest = true;
    } else {
      int a0 = c.ia, b0c = c.ib, na = 1, nb = 1;
      if (c.la > 0) {
        const int2 cr = *reinterpret_cast<const int2*>(wa + 11);
        a0 = cr.x;
        na = cr.y;
      }
      if (c.lb > 0) {
        const int2 cr = *reinterpret_cast<const int2*>(wb + 11);
        b0c = cr.x;
        nb = cr.y;
      }
      P = Parent{c.pair, a0, b0c, (uint8_t)na, (uint8_t)nb, (uint8_t)(c.la > 0 ? c.la - 1 : 0),
                 (uint8_t)(c.lb > 0 ? c.lb - 1 : 0)};
      flagged = true;
    }
  }
  // per-warp appends: one atomic per warp and list
  const unsigned mr = __ballot_sync(0xffffffffu, rest);
  if (mr) {
    unsigned long long rbase = 0;
    if (lane == 0) rbase = atomicAdd(&out.ctr->resting, (unsigned long long)__popc(mr));
    rbase = __shfl_sync(0xffffffffu, rbase, 0);
    const unsigned long long slot = rbase + __popc(mr & ((1u << lane) - 1u));
    if (rest && slot < out.rest_cap) out.resting[slot] = R;
  }
  const unsigned m = __ballot_sync(0xffffffffu, flagged);
  unsigned long long base = 0;
  if (lane == 0 && m) base = atomicAdd(n_par, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (flagged) par[base + __popc(m & ((1u << lane) - 1u))] = P;
}

#ifndef LTSG_GUIDE
#define LTSG_GUIDE 1  // guided single-feature pre-decision before the exact pass of a static generation
#endif
#ifndef LTSG_GUIDE_EDGES
#define LTSG_GUIDE_EDGES 1  // the guide also ranks the nine edge-edge features
#endif
#ifndef LTSG_GUIDE_CULL
#define LTSG_GUIDE_CULL 1  // rows the guide places above the threshold: certified by one separating direction
#endif
#ifndef LTSG_GUIDE_MINB
#define LTSG_GUIDE_MINB 5
#endif
#ifndef LTSG_GUIDE_THREADS
#define LTSG_GUIDE_THREADS 128
#endif
#ifndef LTSG_GUIDE_GRID
#define LTSG_GUIDE_GRID 2  // persistent grid: blocks per resident block slot
#endif
constexpr int kGuideThreads = LTSG_GUIDE_THREADS;

// One exact feature of ccd._feature_distances (ccd.py:135-153), squared,
// from the world records: feature k as numbered by Guide.  The operands are
// the ones feature_dist_sq passes (edges e_k = v[k+1] - v[k]; ab = e0,
// ac = v2 - v0 = -e2 exactly, bc = e1), so the value is bit for bit the
// reference's value of that feature.
__device__ __forceinline__ double one_feature_sq(const double* wa, const double* wb, int k) {
  auto ld = [](const double* p) { return V3{__ldg(p), __ldg(p + 1), __ldg(p + 2)}; };
  if (k < 6) {
    const double* pp = (k < 3 ? wa + 3 * k : wb + 3 * (k - 3));
    const double* tt = k < 3 ? wb : wa;
    const V3 p = ld(pp), a = ld(tt), b = ld(tt + 3), c = ld(tt + 6);
    return point_triangle_sq<false, false>(p, a, b, c, b - a, c - a, c - b);
  }
  const int i = (k - 6) / 3, j = (k - 6) % 3;
  const V3 p1 = ld(wa + 3 * i), q1 = ld(wa + 3 * (i == 2 ? 0 : i + 1));
  const V3 p2 = ld(wb + 3 * j), q2 = ld(wb + 3 * (j == 2 ? 0 : j + 1));
  const V3 u = q1 - p1, w = q2 - p2;
  return segment_segment_sq<false>(p1, u, dot_simd(u, u), p2, w, dot_simd(w, w));
}

// Guided pre-decision of a static generation, one thread per frontier row.
// The FP32 guide (bound32.cuh) names the feature most likely to be the
// row's minimum; that one feature is evaluated with the reference's FP64
// arithmetic, and a row whose exact feature distance is at or below the
// row's threshold is decided: the reference's minimum over 15 features is
// at most this feature (sqrt is monotone and correctly rounded, so
// sqrt(d_k^2) <= T implies sqrt(min d^2) <= T).  Decided rows act here
// (resting record / flagged parent); the others are compacted, one atomic
// per warp, into `rest` for the exact 15-feature pass.  The guide never
// decides anything by itself, so a wrong guess only costs time.
__global__ void __launch_bounds__(kGuideThreads, LTSG_GUIDE_MINB)
k_guide_static(const Cand* __restrict__ front, int64_t n, const PairInfo* __restrict__ pairs,
               const double* __restrict__ world, const int64_t* __restrict__ woff, ScreenOut out,
               Parent* __restrict__ par, unsigned long long* n_par, Cand* __restrict__ rest,
               unsigned long long* n_rest) {
  if (out.n_in) n = (int64_t)min(*out.n_in, out.next_cap);
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n > 0) atomicAdd(&out.ctr->screen_exact, (unsigned long long)n);
  const int64_t n_warps = (n + 31) / 32;
  const int wpb = kGuideThreads / 32;
  unsigned long long decided = 0;
  for (int64_t wi = blockIdx.x * (int64_t)wpb + (threadIdx.x >> 5); wi < n_warps; wi += (int64_t)gridDim.x * wpb) {
    const int64_t ci = wi * 32 + lane;
    bool hit = false, miss = false;
    Cand c{};
    if (ci < n) {
      c = front[ci];
      const double* wa = world + (size_t)c.ia * kWorld;
      const double* wb = world + (size_t)c.ib * kWorld;
      const double h = add(__ldg(wa + 9), __ldg(wb + 9));
      const double T = (c.la == 0 && c.lb == 0) ? add(h, kRestSlop) : h;
      const Guide g = feature_guide<LTSG_GUIDE_EDGES != 0>(wa, wb);
      const float Tf = (float)T;
      if (g.k >= 0) {
        if (g.d2 <= Tf * Tf * 1.002f) {
          hit = __dsqrt_rn(one_feature_sq(wa, wb, g.k)) <= T;
        } else if (LTSG_GUIDE_CULL) {
          // certainly above the threshold: nothing to record for this row
          miss = direction_cull(wa, wb, guide_direction(wa, wb, g.k), add(h, kRestSlop));
        }
      }
    }
    decided += hit || miss;
    static_row_hit(hit, ci, front, pairs, world, woff, out, par, n_par, lane);
    const bool pend = ci < n && !hit && !miss;
    const unsigned m = __ballot_sync(0xffffffffu, pend);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(n_rest, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (pend) rest[base + __popc(m & ((1u << lane) - 1u))] = c;
  }
  for (int o = 16; o > 0; o >>= 1) decided += __shfl_xor_sync(0xffffffffu, decided, o);
  if (lane == 0 && decided) atomicAdd(&out.ctr->bound_rows, decided);
}

// Exact pass of a static generation.  The frontier holds only rows that
// survived the certified culls (and, with LTSG_GUIDE, the guided
// pre-decision), so every row gets the exact 15-feature distance, one per
// lane, from shared-memory staging.  Fine rows apply the resting test
// (ccd.py:407-409); a flagged coarse row (ccd.py:410-411) becomes a Parent,
// appended with one atomic per warp.  The children are generated and culled
// by k_expand_filter at full occupancy.  `count`: add the frontier size to
// the exact-row counter (off when k_guide_static already counted the
// generation's rows).
__global__ void __launch_bounds__(32 * kStaticWarps, LTSG_STATIC_MINB)
k_screen_static(const Cand* __restrict__ front, int64_t n, const PairInfo* __restrict__ pairs,
                const BodyInfo* __restrict__ bodies, const double* __restrict__ world,
                const int64_t* __restrict__ woff, ScreenOut out, Parent* __restrict__ par,
                unsigned long long* n_par, bool count) {
  if (out.n_in) n = (int64_t)min(*out.n_in, out.next_cap);
  extern __shared__ double s_stage[];  // kStaged x (32 * kStaticWarps)
  __shared__ int64_t s_q[kStaticWarps][64];
  const Staged<32 * kStaticWarps> st{s_stage + threadIdx.x};
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int64_t* q = s_q[warp];
  if (count && blockIdx.x == 0 && threadIdx.x == 0 && n > 0)
    atomicAdd(&out.ctr->screen_exact, (unsigned long long)n);
  const int64_t n_warps = (n + 31) / 32;
  unsigned long long decided = 0;
  auto act = [&](bool have, int64_t ci, bool hit) {
    static_row_hit(have && hit, ci, front, pairs, world, woff, out, par, n_par, lane);
  };
  // exact 15-feature distance of a queued row: is it at or below its threshold?
  auto exact_hit = [&](int64_t ci) {
    const Cand c = front[ci];
    const double* wa = world + (size_t)c.ia * kWorld;
    const double* wb = world + (size_t)c.ib * kWorld;
    const double h = add(__ldg(wa + 9), __ldg(wb + 9));
    stage_pair_lite(st, load_world(wa), load_world(wb));
    const double d = __dsqrt_rn(staged_dist_sq_lite(st));
    return (c.la == 0 && c.lb == 0) ? d <= add(h, kRestSlop) : d <= h;
  };
  int nq = 0;
  for (int64_t wi = blockIdx.x * (int64_t)kStaticWarps + warp; wi < n_warps;
       wi += (int64_t)gridDim.x * kStaticWarps) {
    const int64_t ci = wi * 32 + lane;
    // pass 1: the certified FP32 upper bound decides rows certainly at or
    // below the threshold (ccd.py:407 resting, :410-411 flag with dt = 0)
    bool pend = false, hit = false;
    if (ci < n) {
      pend = true;
#if LTSG_BOUND
      const Cand c = front[ci];
      const double* wa = world + (size_t)c.ia * kWorld;
      const double* wb = world + (size_t)c.ib * kWorld;
      if (__ldg(wa + 15) >= 0.0 && __ldg(wb + 15) >= 0.0) {
        const double h = add(__ldg(wa + 9), __ldg(wb + 9));
        const double T = (c.la == 0 && c.lb == 0) ? add(h, kRestSlop) : h;
        double ub, margin;
        if (feature_ub(load_world(wa), load_world(wb), &ub, &margin) && ub + margin <= T) {
          pend = false;
          hit = true;
        }
      }
#endif
    }
    decided += hit;
    act(hit, ci, true);
    // pass 2: the undecided rows, queued per warp, exact 32 at a time
    const unsigned m = __ballot_sync(0xffffffffu, pend);
    if (pend) q[nq + __popc(m & ((1u << lane) - 1u))] = ci;
    nq += __popc(m);
    __syncwarp();
    if (nq >= 32) {
      const int64_t x = q[lane];
      act(true, x, exact_hit(x));
      __syncwarp();
      if (lane < nq - 32) q[lane] = q[32 + lane];
      nq -= 32;
      __syncwarp();
    }
  }
  if (nq > 0) {
    const bool have = lane < nq;
    const int64_t x = have ? q[lane] : 0;
    act(have, x, have && exact_hit(x));
  }
  for (int o = 16; o > 0; o >>= 1) decided += __shfl_xor_sync(0xffffffffu, decided, o);
  if (lane == 0 && decided) atomicAdd(&out.ctr->bound_rows, decided);
}

// Children of the flagged rows of one static generation (ccd.py:418-427),
// one thread per child slot (fan = max_children^2 slots per parent): every
// child is a test (counted here); the certified sphere cull, then the
// separating-axis cull on the block-compacted sphere survivors, settle
// most of them, and the rest are appended (one atomic per block
// iteration) as the next generation's exact frontier.
#ifndef LTSG_EXP_GRID
#define LTSG_EXP_GRID 4
#endif
constexpr int kExpThreads = 256;
constexpr int kExpWarps = kExpThreads / 32;
// Each warp works alone (no block barriers, so the load latency of one warp
// overlaps the work of the others): 32 child slots per step through the
// sphere cull into a per-warp queue; every 32 queued rows get the SAT cull
// with all lanes busy; survivors collect in a per-warp output buffer that
// is flushed 64 at a time with one atomic.
__global__ void __launch_bounds__(kExpThreads, 4)
k_expand_filter(const Parent* __restrict__ par, const unsigned long long* n_par, unsigned long long par_cap,
                int fan, const double* __restrict__ world, const double* __restrict__ wsph, Cand* __restrict__ next,
                unsigned long long next_cap, unsigned long long* n_out, Counters* ctr) {
  const int64_t npar = (int64_t)min(*n_par, par_cap);
  const int64_t total = npar * fan;
  __shared__ Cand s_q[kExpWarps][64];
  __shared__ Cand s_o[kExpWarps][96];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  Cand* q = s_q[warp];
  Cand* o = s_o[warp];
  const unsigned lt = (1u << lane) - 1u;
  int nq = 0, no = 0;
  unsigned long long rows = 0;
  auto flush = [&](int cnt) {  // warp-uniform: write the first cnt buffered rows
    unsigned long long base = 0;
    if (lane == 0 && cnt) base = atomicAdd(n_out, (unsigned long long)cnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int k = lane; k < cnt; k += 32)
      if (base + k < next_cap) next[base + k] = o[k];
    __syncwarp();
    for (int k = cnt + lane; k < no; k += 32) o[k - cnt] = o[k];  // keep the rest (no - cnt < 32)
    __syncwarp();
    no -= cnt;
  };
  auto sat_step = [&](int m) {  // SAT cull of the top m queued rows, survivors to the output buffer
    bool keep = false;
    Cand c{};
    if (lane < m) {
      c = q[nq - m + lane];
      const double* pa = world + (size_t)c.ia * kWorld;
      const double* pb = world + (size_t)c.ib * kWorld;
      keep = !sat_cull(pa, pb, add(add(__ldg(pa + 9), __ldg(pb + 9)), kRestSlop));
    }
    const unsigned mk = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) o[no + __popc(mk & lt)] = c;
    __syncwarp();
    nq -= m;
    no += __popc(mk);
    if (no >= 64) flush(64);
  };
  // The slot -> parent mapping uses 32-bit division (total < 2^32 for any
  // workspace that fits), and the next iteration's parent record is loaded
  // before this iteration's child spheres are tested.
  const int64_t stride = (int64_t)gridDim.x * kExpThreads;
  const bool small = total < ((int64_t)1 << 32);
  auto parent_of = [&](int64_t t, int* j) -> int64_t {
    int64_t pi;
    if (small) {
      const uint32_t tt = (uint32_t)t, f = (uint32_t)fan, p = tt / f;
      pi = p;
      *j = (int)(tt - p * f);
    } else {
      pi = t / fan;
      *j = (int)(t - pi * fan);
    }
    return pi;
  };
  int64_t t = ((int64_t)blockIdx.x * kExpWarps + warp) * 32 + lane;
  Parent Pn{};
  int jn = 0;
  if (t < total) Pn = par[parent_of(t, &jn)];
  for (int64_t t0 = ((int64_t)blockIdx.x * kExpWarps + warp) * 32; t0 < total; t0 += stride) {
    const Parent P = Pn;
    const int j = jn;
    const bool live = t < total;
    t += stride;
    if (t < total) Pn = par[parent_of(t, &jn)];  // prefetch
    bool keep = false;
    Cand c{};
    if (live) {
      const int nb = P.nb;
      if (j < (int)P.na * nb) {
        ++rows;
        const int k = nb == 4 ? (j >> 2) : (nb == 2 ? (j >> 1) : j / nb);
        c = Cand{P.pair, P.a0 + k, P.b0 + (j - k * nb), (int16_t)P.la, (int16_t)P.lb, 0.0};
        keep = !static_child_cull(wsph, c.ia, c.ib);
      }
    }
    const unsigned mk = __ballot_sync(0xffffffffu, keep);
    if (keep) q[nq + __popc(mk & lt)] = c;
    __syncwarp();
    nq += __popc(mk);
    if (nq >= 32) sat_step(32);
  }
  if (nq > 0) sat_step(nq);
  if (no > 0) flush(no);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) rows += __shfl_xor_sync(0xffffffffu, rows, off);
  if (lane == 0 && rows) atomicAdd(&ctr->rows, rows);
}

// ---------------------------------------------------------------- zoom

constexpr int kZoomQueue = 512;  // pending intervals per entry on the first pass
constexpr int kZoomWarps = 4;

struct Interval {
  double a, b;
};

// ccd._isolate_crossings (ccd.py:242-308), one warp per entry.  The
// intervals of a round are processed in order, each sampled at 17 points by
// lanes 0..16; once a bracket exists, intervals starting at or after its lo
// are skipped (ccd.py:278-279), exactly as the reference's sequential loop.
// The reference's pending list is unbounded; here each warp has two queues
// of `qcap` intervals.  An entry that would exceed them is abandoned without
// output and appended to `spill`; the host re-runs the spilled entries
// (`sel`) with a queue 16x larger, until none spills.
__global__ void __launch_bounds__(32 * kZoomWarps)
k_zoom(const Entry* __restrict__ entries, int64_t n, const int64_t* __restrict__ sel,
       const PairInfo* __restrict__ pairs, const BodyInfo* __restrict__ bodies, const double* __restrict__ tris,
       Interval* __restrict__ queue, int qcap, int64_t* __restrict__ spill, Bracket* brackets, Counters* ctr) {
  __shared__ double s_grid[kZoomWarps][kZoomSamples + 1];
  __shared__ double s_stage[kStaged * 32 * kZoomWarps];
  const Staged<32 * kZoomWarps> st{s_stage + threadIdx.x};
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x * (int64_t)kZoomWarps + warp;
  Interval* q0 = queue + gw * 2 * (int64_t)qcap;
  Interval* q1 = q0 + qcap;
  double* grid = s_grid[warp];
  for (int64_t e = gw; e < n; e += (int64_t)gridDim.x * kZoomWarps) {
    const int64_t ei = sel ? sel[e] : e;
    const Entry en = entries[ei];
    const PairInfo p = pairs[en.pair];
    const BodyInfo& A = bodies[p.ba];
    const BodyInfo& B = bodies[p.bb];
    Interval* cur = q0;
    Interval* nxt = q1;
    int n_cur = 1;
    if (lane == 0) cur[0] = Interval{en.lo, en.hi};
    __syncwarp();
    bool have = false;
    double blo = 0.0, bhi = 0.0;
    unsigned long long ref_rows = 0, exec_rows = 0;
    bool overflow = false;
    for (int round = 0; round < 64 && n_cur > 0 && !overflow; ++round) {
      ref_rows += (unsigned long long)n_cur * kZoomSamples;
      int n_nxt = 0;
      for (int iv = 0; iv < n_cur; ++iv) {
        const Interval I = cur[iv];
        if (lane < kZoomSamples) grid[lane] = linspace_at(I.a, I.b, kZoomSamples, lane);
        __syncwarp();
        const bool skip = have && grid[0] >= blo;
        if (!skip) {
          double d = 0.0;
          if (lane < kZoomSamples) d = row_distance(st, tris, A, B, 0, en.ia, 0, en.ib, grid[lane]);
          exec_rows += kZoomSamples;
          const double slack = mul(mul(0.5, en.speed), sub(grid[1], grid[0]));
          const unsigned below = __ballot_sync(0xffffffffu, lane < kZoomSamples && d <= en.h);
          int cut = kZoomSamples;
          if (below) {
            const int j = __ffs(below) - 1;
            blo = j > 0 ? grid[j - 1] : grid[0];
            bhi = grid[j];
            have = true;
            cut = j;
          }
          if (slack > kGrazeTol) {
            const unsigned flags = __ballot_sync(0xffffffffu, lane < cut && d <= add(en.h, slack));
            if (lane == 0) {
              int k = 0;
              while (k < cut) {
                if (!((flags >> k) & 1u)) { ++k; continue; }
                int ke = k;
                while (ke + 1 < cut && ((flags >> (ke + 1)) & 1u)) ++ke;
                const double sa = grid[k > 0 ? k - 1 : 0];
                const double sb = grid[ke + 1 < cut - 1 ? ke + 1 : cut - 1];
                if (sb > sa) {
                  if (n_nxt < qcap) nxt[n_nxt] = Interval{sa, sb}; else overflow = true;
                  ++n_nxt;
                }
                k = ke + 1;
              }
            }
            n_nxt = __shfl_sync(0xffffffffu, n_nxt, 0);
            overflow = __shfl_sync(0xffffffffu, overflow, 0);
          }
        }
        __syncwarp();
      }
      Interval* t = cur;
      cur = nxt;
      nxt = t;
      n_cur = n_nxt < qcap ? n_nxt : qcap;
    }
    if (lane == 0 && overflow) {
      spill[atomicAdd(&ctr->overflow, 1ULL)] = ei;  // re-run with a larger queue
    } else if (lane == 0) {
      atomicAdd(&ctr->zoom_rows, ref_rows);
      atomicAdd(&ctr->zoom_exec, exec_rows);
      if (have) {
        const unsigned long long slot = atomicAdd(&ctr->brackets, 1ULL);
        brackets[slot] = Bracket{en.pair, en.ia, en.ib, 0, blo, bhi, en.h};
      }
    }
    __syncwarp();
  }
}

// ccd._batched_bisect (ccd.py:311-318): 52 halvings, returns hi.
__global__ void k_bisect(const Bracket* __restrict__ br, int64_t n, const PairInfo* __restrict__ pairs,
                         const BodyInfo* __restrict__ bodies, const double* __restrict__ tris,
                         Cross* cross, unsigned long long cross_base, unsigned long long* tau_min_bits) {
  __shared__ double s_stage[kStaged * 64];
  const Staged<64> st{s_stage + threadIdx.x};
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Bracket b = br[i];
  const PairInfo p = pairs[b.pair];
  const BodyInfo& A = bodies[p.ba];
  const BodyInfo& B = bodies[p.bb];
  double lo = b.lo, hi = b.hi;
  for (int it = 0; it < kBisectIters; ++it) {
    const double mid = mul(0.5, add(lo, hi));
    if (row_distance(st, tris, A, B, 0, b.ia, 0, b.ib, mid) <= b.h) hi = mid; else lo = mid;
  }
  cross[cross_base + i] = Cross{b.pair, b.ia, b.ib, 1, hi, b.h};
  // tau >= 0, so the IEEE bit pattern orders like the value
  atomicMin(tau_min_bits + p.problem, (unsigned long long)__double_as_longlong(hi));
}

// ---------------------------------------------------------------- finalize

// 1 in *flag when any problem has a nonzero step (the batch is not static)
__global__ void k_any_moving(const double* __restrict__ problem_dt, int n, int32_t* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool moving = i < n && problem_dt[i] != 0.0;
  if (__any_sync(0xffffffffu, moving) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void k_init_problems(unsigned long long* tau_min_bits, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tau_min_bits[i] = 0x7ff0000000000000ULL;  // +inf
}

// Shared bound, effective step, collision (ccd.py:459-471).  Crossings are
// visited in ascending tau by the reference, so its bound is min(dt, min tau).
__global__ void k_finalize(const unsigned long long* tau_min_bits, const double* problem_dt, int n,
                           double widen, double* dt_out, double* first_out, int32_t* coll_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dt = problem_dt[i];
  const double tmin = __longlong_as_double((long long)tau_min_bits[i]);
  const double bound = tmin < dt ? tmin : dt;
  const bool collision = bound < dt;
  double eff = dt;
  if (collision) {
    const double w = mul(bound, add(1.0, widen));
    eff = dt < w ? dt : w;
  }
  dt_out[i] = eff;
  first_out[i] = collision ? bound : 0.0;
  coll_out[i] = collision ? 1 : 0;
}

struct Record {
  int32_t pair, ia, ib, rest;
  double tau, h;
};

// Resting contacts at tau = 0 and crossings with tau <= dt_eff (ccd.py:473-479).
__global__ void k_collect(const RestRec* rest, int64_t n_rest, const Cross* cross, int64_t n_cross,
                          const PairInfo* pairs, const double* dt_eff, Record* out, Counters* ctr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n_rest) {
    const RestRec r = rest[i];
    out[atomicAdd(&ctr->records, 1ULL)] = Record{r.pair, r.ia, r.ib, 1, 0.0, r.h};
  } else if (i < n_rest + n_cross) {
    const Cross c = cross[i - n_rest];
    if (c.tau <= dt_eff[pairs[c.pair].problem])
      out[atomicAdd(&ctr->records, 1ULL)] = Record{c.pair, c.ia, c.ib, 0, c.tau, c.h};
  }
}

// ---------------------------------------------------------------- contacts

struct Soa {
  int32_t* problem;
  int32_t* body_a;
  int32_t* body_b;
  double* position;
  double* normal;
  double* depth;
  double* t;
  int32_t* tri_a;
  int32_t* tri_b;
  double* threshold;
};

__device__ __forceinline__ void soa_copy(const Soa& s, int64_t i, const Soa& d, int64_t j) {
  d.problem[j] = s.problem[i];
  d.body_a[j] = s.body_a[i];
  d.body_b[j] = s.body_b[i];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    d.position[3 * j + c] = s.position[3 * i + c];
    d.normal[3 * j + c] = s.normal[3 * i + c];
  }
  d.depth[j] = s.depth[i];
  d.t[j] = s.t[i];
  d.tri_a[j] = s.tri_a[i];
  d.tri_b[j] = s.tri_b[i];
  d.threshold[j] = s.threshold[i];
}

// ccd._make_contact (ccd.py:183-213), one thread per record.
__global__ void k_contacts(const Record* recs, int64_t n, const PairInfo* pairs, const BodyInfo* bodies,
                           const double* tris, const int32_t* tri_orig, const double* tbase, Soa o,
                           unsigned long long* key) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Record r = recs[i];
  const PairInfo p = pairs[r.pair];
  const BodyInfo& A = bodies[p.ba];
  const BodyInfo& B = bodies[p.bb];
  const Tri ta = world_at(A.m, rec(tris, A, 0, r.ia), r.tau);
  const Tri tb = world_at(B.m, rec(tris, B, 0, r.ib), r.tau);
  V3 pa, pb;
  const double dist = closest_feature(ta, tb, &pa, &pb);
  V3 pos = scale(pa + pb, 0.5);
  const V3 na = face_normal(ta);
  const V3 nb = face_normal(tb);
  if (fabs(dot_blas(na, nb)) >= kParallelCos) {
    V3 mid;
    if (overlap_centroid(ta, tb, na, &mid)) pos = mid;
  }
  V3 nrm;
  if (dist > 1e-9) {
    const V3 d = pa - pb;
    nrm = V3{dv(d.x, dist), dv(d.y, dist), dv(d.z, dist)};
  } else {
    nrm = nb;
    if (dot_blas(nrm, mean3(ta) - mean3(tb)) < 0.0) nrm = neg(nrm);
  }
  const double depth_raw = sub(r.h, dist);
  const double t0 = tbase[p.problem];
  o.problem[i] = p.problem;
  o.body_a[i] = A.id;
  o.body_b[i] = B.id;
  o.position[3 * i] = pos.x;
  o.position[3 * i + 1] = pos.y;
  o.position[3 * i + 2] = pos.z;
  o.normal[3 * i] = nrm.x;
  o.normal[3 * i + 1] = nrm.y;
  o.normal[3 * i + 2] = nrm.z;
  o.depth[i] = depth_raw > 0.0 ? depth_raw : 0.0;  // max(0.0, h - dist)
  o.t[i] = r.rest ? t0 : add(t0, r.tau);
  o.tri_a[i] = tri_orig[A.level_off[0] + r.ia];
  o.tri_b[i] = tri_orig[B.level_off[0] + r.ib];
  o.threshold[i] = r.h;
  key[i] = ((unsigned long long)(uint32_t)p.problem << 32) | (uint32_t)p.group;
}

// ---------------------------------------------------------------- fusion

__device__ __forceinline__ double round9(double x) {  // round(np.float64, 9) = rint(x*1e9)/1e9
  return dv(rint(mul(x, 1e9)), 1e9);
}

// Sort key of ccd.py:541-542: (t, round9(x), round9(y), round9(z), tri_a, tri_b).
__device__ __forceinline__ bool key_less(const Soa& o, int64_t a, int64_t b) {
  if (o.t[a] != o.t[b]) return o.t[a] < o.t[b];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double ra = round9(o.position[3 * a + k]), rb = round9(o.position[3 * b + k]);
    if (ra != rb) return ra < rb;
  }
  if (o.tri_a[a] != o.tri_a[b]) return o.tri_a[a] < o.tri_a[b];
  return o.tri_b[a] < o.tri_b[b];
}



// filter_contacts, one block per (problem, body pair) group of at most
// kFuseCap records, staged in shared memory: keys and positions are loaded
// once, the stable sort is a parallel rank sort, the "within max(threshold)"
// adjacency is a bit matrix built by all threads, and one thread replays the
// reference's union-find over it (ccd.py:543-555) so roots -- and therefore
// the output order -- are identical.  Larger groups go to k_fuse_large.
constexpr int kFuseCap = 256;
constexpr int kFuseWords = kFuseCap / 32;
constexpr int kFuseThreads = 256;

// norm_blas(w) <= r, decided exactly: fl(sqrt(s)) <= r  <=>  s <= r*r up to a
// few ulps, so the square root is only evaluated inside that band.
// Outside it: s < fl(r*r)(1 - 2^-49) implies s < r^2, hence sqrt(s) < r;
// s > fl(r*r)(1 + 2^-49) implies sqrt(s) > r (1 + 2^-52) >= r + ulp(r)/2,
// which rounds above r.
__device__ __forceinline__ bool norm_le(V3 w, double r) {
  const double s = dot_blas(w, w);
  const double p = r * r;
  if (p > 1e-290 && p < 1e290) {
    if (s < p * (1.0 - 0x1p-49)) return true;
    if (s > p * (1.0 + 0x1p-49)) return false;
  }
  return __dsqrt_rn(s) <= r;
}

struct FuseKey {
  double t, r0, r1, r2;
  int32_t ta, tb;
};

__device__ __forceinline__ bool fkey_less(const FuseKey& a, const FuseKey& b) {
  if (a.t != b.t) return a.t < b.t;
  if (a.r0 != b.r0) return a.r0 < b.r0;
  if (a.r1 != b.r1) return a.r1 < b.r1;
  if (a.r2 != b.r2) return a.r2 < b.r2;
  if (a.ta != b.ta) return a.ta < b.ta;
  return a.tb < b.tb;
}

__global__ void __launch_bounds__(kFuseThreads, 4)
k_fuse_block(Soa o, int64_t* __restrict__ idx, const int64_t* __restrict__ g_off, int64_t n_groups,
             int64_t n_total, Soa f, int64_t* g_fused, int32_t* prob_count, int32_t* big_list,
             int32_t* big_count) {
  __shared__ FuseKey s_key[kFuseCap];
  __shared__ int64_t s_gi[kFuseCap];
  __shared__ double s_p[3][kFuseCap];
  __shared__ double s_thr[kFuseCap];
  __shared__ double s_n[3][kFuseCap];
  __shared__ double s_dep[kFuseCap];
  __shared__ double s_tt[kFuseCap];
  __shared__ int32_t s_par[kFuseCap];
  __shared__ int32_t s_slot[kFuseCap];
  __shared__ uint32_t s_adj[kFuseCap * kFuseWords];
  __shared__ int32_t s_nroots;
  __shared__ uint32_t s_lab[kFuseWords];
  const int tid = threadIdx.x;
  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int64_t off = g_off[g];
    const int n = (int)((g + 1 < n_groups ? g_off[g + 1] : n_total) - off);
    if (n > kFuseCap) {
      if (tid == 0) big_list[atomicAdd(big_count, 1)] = (int32_t)g;
      continue;
    }
    int64_t* ix = idx + off;
    __syncthreads();
    for (int i = tid; i < n; i += kFuseThreads) {
      const int64_t a = ix[i];
      FuseKey k;
      k.t = o.t[a];
      k.r0 = round9(o.position[3 * a]);
      k.r1 = round9(o.position[3 * a + 1]);
      k.r2 = round9(o.position[3 * a + 2]);
      k.ta = o.tri_a[a];
      k.tb = o.tri_b[a];
      s_key[i] = k;
    }
    __syncthreads();
    // stable rank sort (ccd.py:541-542): equal keys keep their input order
    for (int i = tid; i < n; i += kFuseThreads) {
      const FuseKey ki = s_key[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const FuseKey kj = s_key[j];
        rank += (fkey_less(kj, ki) || (j < i && !fkey_less(ki, kj))) ? 1 : 0;
      }
      const int64_t a = ix[i];
      s_gi[rank] = a;
      s_p[0][rank] = o.position[3 * a];
      s_p[1][rank] = o.position[3 * a + 1];
      s_p[2][rank] = o.position[3 * a + 2];
      s_thr[rank] = o.threshold[a];
      s_n[0][rank] = o.normal[3 * a];
      s_n[1][rank] = o.normal[3 * a + 1];
      s_n[2][rank] = o.normal[3 * a + 2];
      s_dep[rank] = o.depth[a];
      s_tt[rank] = o.t[a];
    }
    __syncthreads();
    for (int r = tid; r < n; r += kFuseThreads) ix[r] = s_gi[r];  // canonical raw order
    // adjacency bit matrix, upper triangle: |p_i - p_j| <= max(thr_i, thr_j) (ccd.py:551-555)
    const int words = (n + 31) / 32;
    for (int w = tid; w < n * words; w += kFuseThreads) {
      const int row = w / words, word = w % words;
      const V3 pi{s_p[0][row], s_p[1][row], s_p[2][row]};
      const double ti = s_thr[row];
      uint32_t bits = 0;
      for (int b = 0; b < 32; ++b) {
        const int j = word * 32 + b;
        if (j <= row || j >= n) continue;
        const V3 pj{s_p[0][j], s_p[1][j], s_p[2][j]};
        if (norm_le(pi - pj, fmax(ti, s_thr[j]))) bits |= 1u << b;
      }
      s_adj[row * kFuseWords + word] = bits;
    }
    __syncthreads();
    // Union-find of ccd.py:543-555 replayed row by row: processing row i
    // attaches the set of every neighbour j > i under find(i), so after the
    // row every such set carries i's representative.  Keeping the current
    // representative of every element (quick-find) gives the same
    // representatives as the reference's parent forest, with each row done
    // by all threads: collect the neighbours' labels, relabel in parallel.
    for (int i = tid; i < n; i += kFuseThreads) s_par[i] = i;
    for (int w = tid; w < kFuseWords; w += kFuseThreads) s_lab[w] = 0u;
    __syncthreads();
    for (int i = 0; i < n; ++i) {
      const int ri = s_par[i];
      bool any = false;
      for (int j = i + 1 + tid; j < n; j += kFuseThreads) {
        if ((s_adj[i * kFuseWords + (j >> 5)] >> (j & 31)) & 1u) {
          const int rj = s_par[j];
          if (rj != ri) {
            atomicOr(&s_lab[rj >> 5], 1u << (rj & 31));
            any = true;
          }
        }
      }
      if (!__syncthreads_or(any)) continue;
      for (int k = tid; k < n; k += kFuseThreads) {
        const int rk = s_par[k];
        if ((s_lab[rk >> 5] >> (rk & 31)) & 1u) s_par[k] = ri;
      }
      __syncthreads();
      for (int w = tid; w < kFuseWords; w += kFuseThreads) s_lab[w] = 0u;
      __syncthreads();
    }
    if (tid == 0) {
      int nr = 0;
      for (int i = 0; i < n; ++i)
        if (s_par[i] == i) s_slot[i] = nr++;
      s_nroots = nr;
    }
    __syncthreads();
    for (int r = tid; r < n; r += kFuseThreads) {
      if (s_par[r] != r) continue;
      V3 ps{0, 0, 0}, ns{0, 0, 0};
      int cnt = 0, rep = -1, first = -1;
      double dmax = 0.0, tmin = 0.0, thr = 0.0;
      for (int i = 0; i < n; ++i) {  // members in ascending sorted order (ccd.py:557-558)
        if (s_par[i] != r) continue;
        const V3 pp{s_p[0][i], s_p[1][i], s_p[2][i]};
        const V3 nn{s_n[0][i], s_n[1][i], s_n[2][i]};
        const double da = s_dep[i], ta = s_tt[i], tha = s_thr[i];
        if (cnt == 0) {
          first = i;
          rep = i;
          ps = pp;
          ns = nn;
          dmax = da;
          tmin = ta;
          thr = tha;
        } else {
          ps = ps + pp;  // np.mean / np.sum over axis 0: sequential
          ns = ns + nn;
          if (da > dmax) dmax = da;
          if (ta < tmin) tmin = ta;
          if (tha > thr) thr = tha;
          // min(group, key=(t, -depth)): the first strictly smaller wins
          if (ta < s_tt[rep] || (ta == s_tt[rep] && -da < -s_dep[rep])) rep = i;
        }
        ++cnt;
      }
      const double c = (double)cnt;
      const V3 pos{dv(ps.x, c), dv(ps.y, c), dv(ps.z, c)};
      const double ln = norm_blas(ns);
      V3 nrm;
      if (ln > 1e-12) {
        nrm = V3{dv(ns.x, ln), dv(ns.y, ln), dv(ns.z, ln)};
      } else {
        nrm = V3{s_n[0][first], s_n[1][first], s_n[2][first]};
      }
      const int64_t ra = s_gi[rep];
      const int64_t dst = off + s_slot[r];
      f.problem[dst] = o.problem[ra];
      f.body_a[dst] = o.body_a[ra];
      f.body_b[dst] = o.body_b[ra];
      f.position[3 * dst] = pos.x;
      f.position[3 * dst + 1] = pos.y;
      f.position[3 * dst + 2] = pos.z;
      f.normal[3 * dst] = nrm.x;
      f.normal[3 * dst + 1] = nrm.y;
      f.normal[3 * dst + 2] = nrm.z;
      f.depth[dst] = dmax;
      f.t[dst] = tmin;
      f.tri_a[dst] = o.tri_a[ra];
      f.tri_b[dst] = o.tri_b[ra];
      f.threshold[dst] = thr;
    }
    if (tid == 0) {
      g_fused[g] = s_nroots;
      if (n > 0) atomicAdd(prob_count + o.problem[ix[0]], s_nroots);
    }
  }
}

// Groups larger than kFuseCap: one 512-thread block per group, the same
// steps as k_fuse_block with the per-record arrays and the adjacency bit
// matrix in global scratch (records stay in their group's slot range).
constexpr int kFuseLargeThreads = 512;

__global__ void __launch_bounds__(kFuseLargeThreads)
k_fuse_large(Soa o, int64_t* __restrict__ idx, const int64_t* __restrict__ g_off, int64_t n_groups,
             int64_t n_total, Soa f, int64_t* g_fused, int32_t* prob_count, const int32_t* big_list,
             const int64_t* adj_off, FuseKey* key, int64_t* gi, double* pos, double* thrs, int32_t* par,
             int32_t* slot, uint32_t* adj_all) {
  __shared__ int32_t s_nroots;
  const int tid = threadIdx.x;
  const int64_t g = big_list[blockIdx.x];
  const int64_t off = g_off[g];
  const int n = (int)((g + 1 < n_groups ? g_off[g + 1] : n_total) - off);
  int64_t* ix = idx + off;
  FuseKey* k_ = key + off;
  int64_t* gi_ = gi + off;
  double* px = pos + 3 * off;
  double* th = thrs + off;
  int32_t* pr = par + off;
  int32_t* sl = slot + off;
  const int words = (n + 31) / 32;
  uint32_t* adj = adj_all + adj_off[blockIdx.x];
  for (int i = tid; i < n; i += kFuseLargeThreads) {
    const int64_t a = ix[i];
    FuseKey k;
    k.t = o.t[a];
    k.r0 = round9(o.position[3 * a]);
    k.r1 = round9(o.position[3 * a + 1]);
    k.r2 = round9(o.position[3 * a + 2]);
    k.ta = o.tri_a[a];
    k.tb = o.tri_b[a];
    k_[i] = k;
  }
  __syncthreads();
  for (int i = tid; i < n; i += kFuseLargeThreads) {
    const FuseKey ki = k_[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const FuseKey kj = k_[j];
      rank += (fkey_less(kj, ki) || (j < i && !fkey_less(ki, kj))) ? 1 : 0;
    }
    const int64_t a = ix[i];
    gi_[rank] = a;
    px[3 * rank] = o.position[3 * a];
    px[3 * rank + 1] = o.position[3 * a + 1];
    px[3 * rank + 2] = o.position[3 * a + 2];
    th[rank] = o.threshold[a];
  }
  __syncthreads();
  for (int r = tid; r < n; r += kFuseLargeThreads) ix[r] = gi_[r];
  for (int64_t w = tid; w < (int64_t)n * words; w += kFuseLargeThreads) {
    const int row = (int)(w / words), word = (int)(w % words);
    const V3 pi{px[3 * row], px[3 * row + 1], px[3 * row + 2]};
    const double ti = th[row];
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int j = word * 32 + b;
      if (j <= row || j >= n) continue;
      const V3 pj{px[3 * j], px[3 * j + 1], px[3 * j + 2]};
      if (norm_le(pi - pj, fmax(ti, th[j]))) bits |= 1u << b;
    }
    adj[(int64_t)row * words + word] = bits;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < n; ++i) pr[i] = i;
    auto find = [&](int x) {  // path halving, as the reference's find (ccd.py:545-549)
      while (pr[x] != x) {
        pr[x] = pr[pr[x]];
        x = pr[x];
      }
      return x;
    };
    for (int i = 0; i < n; ++i) {
      const int ri = find(i);
      for (int word = i / 32; word < words; ++word) {
        uint32_t bits = adj[(int64_t)i * words + word];
        while (bits) {
          const int j = word * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          pr[find(j)] = ri;
        }
      }
    }
    int nr = 0;
    for (int i = 0; i < n; ++i) pr[i] = find(i);
    for (int i = 0; i < n; ++i)
      if (pr[i] == i) sl[i] = nr++;
    s_nroots = nr;
  }
  __syncthreads();
  for (int r = tid; r < n; r += kFuseLargeThreads) {
    if (pr[r] != r) continue;
    V3 ps{0, 0, 0}, ns{0, 0, 0};
    int cnt = 0;
    int64_t rep = -1, first = -1;
    double dmax = 0.0, tmin = 0.0, thr = 0.0;
    for (int i = 0; i < n; ++i) {
      if (pr[i] != r) continue;
      const int64_t a = gi_[i];
      const V3 pp{px[3 * i], px[3 * i + 1], px[3 * i + 2]};
      const V3 nn{o.normal[3 * a], o.normal[3 * a + 1], o.normal[3 * a + 2]};
      const double da = o.depth[a], ta = o.t[a], tha = o.threshold[a];
      if (cnt == 0) {
        first = a;
        rep = a;
        ps = pp;
        ns = nn;
        dmax = da;
        tmin = ta;
        thr = tha;
      } else {
        ps = ps + pp;
        ns = ns + nn;
        if (da > dmax) dmax = da;
        if (ta < tmin) tmin = ta;
        if (tha > thr) thr = tha;
        if (ta < o.t[rep] || (ta == o.t[rep] && -da < -o.depth[rep])) rep = a;
      }
      ++cnt;
    }
    const double c = (double)cnt;
    const V3 psn{dv(ps.x, c), dv(ps.y, c), dv(ps.z, c)};
    const double ln = norm_blas(ns);
    V3 nrm;
    if (ln > 1e-12) nrm = V3{dv(ns.x, ln), dv(ns.y, ln), dv(ns.z, ln)};
    else nrm = V3{o.normal[3 * first], o.normal[3 * first + 1], o.normal[3 * first + 2]};
    const int64_t dst = off + sl[r];
    f.problem[dst] = o.problem[rep];
    f.body_a[dst] = o.body_a[rep];
    f.body_b[dst] = o.body_b[rep];
    f.position[3 * dst] = psn.x;
    f.position[3 * dst + 1] = psn.y;
    f.position[3 * dst + 2] = psn.z;
    f.normal[3 * dst] = nrm.x;
    f.normal[3 * dst + 1] = nrm.y;
    f.normal[3 * dst + 2] = nrm.z;
    f.depth[dst] = dmax;
    f.t[dst] = tmin;
    f.tri_a[dst] = o.tri_a[rep];
    f.tri_b[dst] = o.tri_b[rep];
    f.threshold[dst] = thr;
  }
  if (tid == 0) {
    g_fused[g] = s_nroots;
    atomicAdd(prob_count + o.problem[ix[0]], s_nroots);
  }
}

__global__ void k_compact(Soa f, const int64_t* g_off, const int64_t* g_fused, const int64_t* g_dst,
                          int64_t n_groups, Soa o) {
  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int64_t src = g_off[g], dst = g_dst[g], n = g_fused[g];
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) soa_copy(f, src + k, o, dst + k);
  }
}

__global__ void k_gather(Soa s, const int64_t* idx, int64_t n, Soa d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) soa_copy(s, idx[i], d, i);
}

__global__ void k_heads(const unsigned long long* keys, int64_t n, int64_t* head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  if (i == n) head[n] = 0;
}

__global__ void k_group_table(const int64_t* head, const int64_t* head_scan, int64_t n, int64_t* g_off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && head[i]) g_off[head_scan[i]] = i;
}

__global__ void k_iota(int64_t* x, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}

__global__ void k_widen(const int32_t* a, int64_t* b, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// Exhaustive fine x fine rows as register x broadcast tiles (the roofline
// kernel; ccd._search with exhaustive=True evaluates the same rows,
// ccd.py:385-391).  A work item is (pair, tile of kTileA fine triangles of
// body a, tile of kTileB fine triangles of body b).  Each lane holds one A
// triangle with its per-triangle constants in registers; the B tile is
// staged once in shared memory and every lane of a warp walks it in the
// same order, so each B operand is one broadcast load.  Work items are
// distributed over a persistent grid from a per-pair prefix of item counts.
constexpr int kTileA = 128;
constexpr int kTileB = 32;
#ifndef LTSG_TILE_MINB
#define LTSG_TILE_MINB 6
#endif

constexpr int kTileSmemBytes = (kTileB * kTilePre + kTileA * kTileASlots) * 8;

__global__ void __launch_bounds__(kTileA, LTSG_TILE_MINB)
k_allpairs_tile(const PairInfo* __restrict__ pairs, int64_t n_pairs, const BodyInfo* __restrict__ bodies,
                const double* __restrict__ world, const int64_t* __restrict__ woff,
                const int64_t* __restrict__ item_start, const int64_t* __restrict__ row_start,
                unsigned long long* hits, double* __restrict__ out_dist) {
  extern __shared__ __align__(16) double s_tile[];
  double* sB = s_tile;                       // [kTileB][kTilePre], broadcast reads
  double* sA = s_tile + kTileB * kTilePre;   // [kTilePre][kTileA], one column per lane
  unsigned long long local = 0;
  const int64_t n_items = item_start[n_pairs];
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    int64_t lo = 0, hi = n_pairs;  // last pair k with item_start[k] <= item
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(item_start + mid) <= item) lo = mid; else hi = mid;
    }
    const PairInfo p = pairs[lo];
    const int na = bodies[p.ba].level_size[0], nb = bodies[p.bb].level_size[0];
    const int tiles_b = (nb + kTileB - 1) / kTileB;
    const int64_t local_item = item - item_start[lo];
    const int ta = (int)(local_item / tiles_b), tb = (int)(local_item - (int64_t)ta * tiles_b);
    const int jb0 = tb * kTileB, nbt = min(kTileB, nb - jb0);
    __syncthreads();  // the previous item's tiles are no longer read
    if (threadIdx.x < nbt) {
      const double* wb = world + (size_t)(woff[p.bb] + jb0 + threadIdx.x) * kWorld;
      tri_store(sB + threadIdx.x * kTilePre, tri_reg(load_world(wb), __ldg(wb + 9)));
    }
    const int i = ta * kTileA + threadIdx.x;
    const bool valid = i < na;
    const double* wa = world + (size_t)(woff[p.ba] + (valid ? i : na - 1)) * kWorld;
    const double eps_a = __ldg(wa + 9);
    const TriReg ar = tri_reg(load_world(wa), eps_a);
    const bool a_regular = ar.regular;
    tri_store_soa<kTileA>(sA + threadIdx.x, ar);
    __syncthreads();
    const SmemTri<kTileA> A{sA + threadIdx.x};
    double* od = out_dist ? out_dist + row_start[lo] + (int64_t)(valid ? i : 0) * nb + jb0 : nullptr;
#pragma unroll 1
    for (int j = 0; j < nbt; ++j) {
      const double* t = sB + j * kTilePre;
      const double d = __dsqrt_rn(tile_dist_sq(A, a_regular, t));
      if (valid && d <= add(add(eps_a, t[kTpEps]), kRestSlop)) ++local;
      if (od && valid) od[j] = d;
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(hits, local);
}

// ---------------------------------------------------------------- host side

template <typename T>
static int ws_get(ltsg_workspace* ws, const char* name, size_t count, T** out, bool keep = false) {
  void* p = nullptr;
  LTSG_TRY(ws->get(name, std::max<size_t>(count, 1) * sizeof(T), &p, keep));
  *out = static_cast<T*>(p);
  return LTSG_OK;
}

static int read_ctr(Counters* d, Counters* h, cudaStream_t st) {
  LTSG_CUDA(cudaMemcpyAsync(h, d, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  return LTSG_OK;
}

static int scan_exclusive(ltsg_workspace* ws, const int64_t* in, int64_t* out, int64_t n, cudaStream_t st) {
  size_t tmp = 0;
  LTSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st));
  void* t = nullptr;
  LTSG_TRY(ws->get("cub_tmp", tmp, &t));
  LTSG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, st));
  return LTSG_OK;
}

constexpr int kScreenStageBytes = kStagedLite * 32 * kScreenWarps * sizeof(double);

static int configure_kernels() {
  static int done = 0;
  if (!done) {
    LTSG_CUDA(cudaFuncSetAttribute(k_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, kScreenStageBytes));
    LTSG_CUDA(cudaFuncSetAttribute(k_screen_static, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kStaticStageBytes));
    LTSG_CUDA(cudaFuncSetAttribute(k_allpairs_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemBytes));
    LTSG_CUDA(cudaFuncSetAttribute(k_mexact, cudaFuncAttributeMaxDynamicSharedMemorySize, kMExactStageBytes));
    done = 1;
  }
  return LTSG_OK;
}

static int screen_grid(int64_t n) {
  const int64_t warps = (n + 31) / 32;
  const int64_t blocks = (warps + kScreenWarps - 1) / kScreenWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, 148LL * 32));
}

struct Prepared {
  BodyInfo* bodies;
  PairInfo* pairs;
};

static int validate(const ltsg_scene* sc) {
  if (!sc || sc->n_bodies < 0 || sc->n_pairs < 0 || sc->n_problems < 0 || sc->max_children < 1 ||
      (sc->n_pairs > 0 && (!sc->tris || !sc->body_state || !sc->body_levels || !sc->pair_body ||
                           !sc->pair_problem || !sc->pair_group || !sc->problem_dt ||
                           !sc->problem_tbase || !sc->tri_orig))) {
    set_error("ltsg_search: invalid scene");
    return LTSG_EINVAL;
  }
  return LTSG_OK;
}

static int prepare(const ltsg_scene* sc, ltsg_workspace* ws, cudaStream_t st, Prepared* pr) {
  LTSG_TRY(ws_get(ws, "bodies", (size_t)sc->n_bodies, &pr->bodies));
  LTSG_TRY(ws_get(ws, "pairs", (size_t)sc->n_pairs, &pr->pairs));
  if (sc->n_bodies > 0) {
    k_prep_bodies<<<grid_for(sc->n_bodies, 128), 128, 0, st>>>(sc->body_state, sc->body_levels,
                                                               sc->n_bodies, pr->bodies);
    LTSG_CHECK_LAUNCH();
  }
  if (sc->n_pairs > 0) {
    k_prep_pairs<<<grid_for(sc->n_pairs, 128), 128, 0, st>>>(sc->pair_body, sc->pair_problem,
                                                             sc->pair_group, sc->n_pairs, pr->bodies,
                                                             sc->problem_dt, pr->pairs);
    LTSG_CHECK_LAUNCH();
  }
  return LTSG_OK;
}

static int fuse_stage(ltsg_workspace* ws, cudaStream_t st, Soa ro, unsigned long long* key, int64_t n_rec,
                      int np, int32_t* prob_count, int64_t* prob_count64, ltsg_result* out);

// Device-time accounting of one call: CUDA events on the call's stream.
struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  Timer() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~Timer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  void start(cudaStream_t st) { cudaEventRecord(a, st); }
  void stop(cudaStream_t st) { cudaEventRecord(b, st); }
  double ms() {  // call after the stream has passed `b`
    float m = 0.f;
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&m, a, b);
    return (double)m;
  }
};

// Optional phase trace (env LTSG_TRACE=1): device time and host wall time
// between consecutive marks of one call, printed to stderr.  Diagnostic only.
struct Trace {
  bool on = false;
  cudaStream_t st = nullptr;
  std::vector<const char*> name;
  std::vector<cudaEvent_t> ev;
  std::vector<double> host_us;
  explicit Trace(cudaStream_t s) : st(s) {
    const char* e = getenv("LTSG_TRACE");
    on = e && e[0] == '1';
  }
  static double now_us() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return 1e6 * (double)t.tv_sec + 1e-3 * (double)t.tv_nsec;
  }
  void mark(const char* n) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    name.push_back(n);
    ev.push_back(e);
    host_us.push_back(now_us());
  }
  ~Trace() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back());
    fprintf(stderr, "[ltsg trace] %-14s %10s %10s\n", "phase", "device_ms", "host_ms");
    for (size_t i = 1; i < ev.size(); ++i) {
      float m = 0.f;
      cudaEventElapsedTime(&m, ev[i - 1], ev[i]);
      fprintf(stderr, "[ltsg trace] %-14s %10.3f %10.3f\n", name[i], m, 1e-3 * (host_us[i] - host_us[i - 1]));
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
};

#define LTSG_LAUNCHED() \
  do {                  \
    LTSG_CHECK_LAUNCH(); \
    ++out->launches;    \
  } while (0)

static int run_search(const ltsg_scene* sc, ltsg_result* out, ltsg_workspace* ws, cudaStream_t st) {
  LTSG_TRY(validate(sc));
  LTSG_TRY(configure_kernels());
  const int np = sc->n_problems;
  out->n_fused = out->n_raw = 0;
  out->rows_screen = out->rows_zoom = out->rows_bisect = out->rows_executed = 0;
  out->candidates = 0;
  out->generations = 0;
  out->launches = 0;
  out->ms_screen = out->ms_refine = out->ms_contacts = 0.0;
  out->rows_screen_exact = 0;
  out->rows_bound = 0;
  out->ms_exact = out->ms_expand = 0.0;
  if (np == 0) return LTSG_OK;

  Trace tr(st);
  tr.mark("start");
  Prepared pr{};
  LTSG_TRY(prepare(sc, ws, st, &pr));
  out->launches += 2;
  tr.mark("prepare");
  Timer t_screen, t_refine, t_contacts;
  Counters* d_ctr;
  LTSG_TRY(ws_get(ws, "ctr", 1, &d_ctr));
  LTSG_CUDA(cudaMemsetAsync(d_ctr, 0, sizeof(Counters), st));
  unsigned long long* tau_min;
  LTSG_TRY(ws_get(ws, "tau_min", (size_t)np, &tau_min));
  k_init_problems<<<grid_for(np, 128), 128, 0, st>>>(tau_min, np);
  LTSG_LAUNCHED();

  // ---- static batches: tau = 0 world records, sphere data, culled seeds.
  // Three host decisions are needed before the traversal can be sized: is
  // every step zero, how many world records, how many seed rows.  Their
  // inputs are computed back to back and read with ONE synchronisation.
  bool all_static = false;
  double* world = nullptr;
  double* wsph = nullptr;
  int64_t* woff = nullptr;
  int64_t seed_total = 0;
  int64_t *seed_cnt = nullptr, *seed_off = nullptr;
  if (sc->n_pairs > 0) {
    int32_t* d_moving;
    int64_t* wcnt;
    LTSG_TRY(ws_get(ws, "any_moving", (size_t)1, &d_moving));
    LTSG_TRY(ws_get(ws, "world_cnt", (size_t)sc->n_bodies + 1, &wcnt));
    LTSG_TRY(ws_get(ws, "world_off", (size_t)sc->n_bodies + 1, &woff));
    LTSG_TRY(ws_get(ws, "seed_cnt", (size_t)sc->n_pairs + 1, &seed_cnt));
    LTSG_TRY(ws_get(ws, "seed_off", (size_t)sc->n_pairs + 1, &seed_off));
    LTSG_CUDA(cudaMemsetAsync(d_moving, 0, sizeof(int32_t), st));
    k_any_moving<<<grid_for(np, 128), 128, 0, st>>>(sc->problem_dt, np, d_moving);
    LTSG_LAUNCHED();
    k_world_count<<<grid_for(sc->n_bodies + 1, 128), 128, 0, st>>>(pr.bodies, sc->n_bodies, wcnt);
    LTSG_LAUNCHED();
    LTSG_TRY(scan_exclusive(ws, wcnt, woff, sc->n_bodies + 1, st));
    k_seed_count<<<grid_for(sc->n_pairs, 128), 128, 0, st>>>(pr.pairs, sc->n_pairs, pr.bodies,
                                                             sc->exhaustive, seed_cnt);
    LTSG_LAUNCHED();
    LTSG_CUDA(cudaMemsetAsync(seed_cnt + sc->n_pairs, 0, sizeof(int64_t), st));
    LTSG_TRY(scan_exclusive(ws, seed_cnt, seed_off, sc->n_pairs + 1, st));
    int32_t h_moving = 1;
    int64_t n_world = 0;
    LTSG_CUDA(cudaMemcpyAsync(&h_moving, d_moving, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaMemcpyAsync(&n_world, woff + sc->n_bodies, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaMemcpyAsync(&seed_total, seed_off + sc->n_pairs, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaStreamSynchronize(st));
    all_static = h_moving == 0;
    if (sc->max_children > 255) all_static = false;  // static parents hold 8-bit child counts
    const char* env = getenv("LTSG_NO_STATIC");
    if (env && env[0] == '1') all_static = false;
    if (n_world >= (int64_t)1 << 31) all_static = false;  // world indices are int32 in the candidates
    if (all_static) {
      LTSG_TRY(ws_get(ws, "world", (size_t)std::max<int64_t>(n_world, 1) * (kWorld + kSph), &world));
      wsph = world + (size_t)std::max<int64_t>(n_world, 1) * kWorld;
      k_world_fill<<<(int)std::max<int64_t>(1, std::min<int64_t>((n_world + 127) / 128, 148 * 16)), 128, 0, st>>>(
          pr.bodies, sc->n_bodies, woff, sc->tris, world, wsph);
      LTSG_LAUNCHED();
    } else {
      woff = nullptr;
    }
  }

  tr.mark("world");
  // ---- pose tables for moving batches
  PoseTable poses{nullptr, nullptr, nullptr};
  if (!all_static && sc->n_pairs > 0 && sc->n_bodies > 0) {
    double* cm;
    LTSG_TRY(ws_get(ws, "cull_m", (size_t)sc->n_bodies * kCullM, &cm));
    k_cull_prep<<<grid_for(sc->n_bodies, 128), 128, 0, st>>>(pr.bodies, sc->n_bodies, cm);
    LTSG_LAUNCHED();
    poses.cm = cm;
  }
  if (!all_static && sc->n_pairs > 0 && sc->n_bodies > 0 && !getenv("LTSG_NO_POSES")) {
    const size_t bytes = (size_t)sc->n_bodies * kPoseEntries * kPose * sizeof(double);
    if (bytes <= ws->budget / 4) {
      double *tab, *tdt;
      LTSG_TRY(ws_get(ws, "pose_tab", (size_t)sc->n_bodies * kPoseEntries * kPose, &tab));
      LTSG_TRY(ws_get(ws, "pose_dt", (size_t)sc->n_bodies, &tdt));
      LTSG_CUDA(cudaMemsetAsync(tdt, 0xff, sizeof(double) * sc->n_bodies, st));  // NaN
      k_pose_dt<<<grid_for(sc->n_pairs, 128), 128, 0, st>>>(pr.pairs, sc->n_pairs, tdt);
      LTSG_LAUNCHED();
      k_pose_fill<<<148 * 16, 128, 0, st>>>(pr.bodies, sc->n_bodies, tdt, tab);
      LTSG_LAUNCHED();
      poses.tab = tab;
      poses.tdt = tdt;
    }
  }

  // ---- traversal: seeds (ccd.py:385-391) and generations (ccd.py:393-446).
  // Async mode enqueues every generation back to back (frontier sizes stay
  // on the device, buffers are sized from the workspace's history) and
  // checks once at the end; on any overflow the traversal re-runs in sync
  // mode, which reads each frontier size back and grows buffers as needed.
  tr.mark("poses+seedcnt");
  constexpr int kMaxGen = 2 * kMaxLevels;
  unsigned long long *gen_cnt, *x_cnt;
  LTSG_TRY(ws_get(ws, "gen_cnt", kMaxGen + 1, &gen_cnt));
  LTSG_TRY(ws_get(ws, "x_cnt", 2 * (kMaxGen + 1), &x_cnt));  // static: flagged parents per generation
  const int64_t fan = (int64_t)sc->max_children * sc->max_children;
  size_t rest_cap = std::max<size_t>(1 << 16, ws->hint_rest), entry_cap = std::max<size_t>(1 << 14, ws->hint_entries),
         cross_cap = std::max<size_t>(1 << 14, ws->hint_cross);
  RestRec* resting;
  Entry* entries;
  Cross* cross;
  Counters h{};
  Cand* front = nullptr;

  // moving batches: rows surviving the culls, per generation (k_mscreen -> k_mexact -> k_mdecide)
  const bool legacy_moving = getenv("LTSG_MOVING_LEGACY") != nullptr;
  ExactRow* mrows = nullptr;
  size_t mrows_cap = 0;
  size_t n_timed = 0;  // generations timed with event triples (exact, expand / decide)
  auto static_times = [&]() -> int {  // call once the stream has passed every recorded event
    out->ms_exact = out->ms_expand = 0.0;
    for (size_t g = 0; g < n_timed; ++g) {
      float a = 0.f, b = 0.f;
      LTSG_CUDA(cudaEventSynchronize(ws->event(3 * g + 2)));
      LTSG_CUDA(cudaEventElapsedTime(&a, ws->event(3 * g), ws->event(3 * g + 1)));
      LTSG_CUDA(cudaEventElapsedTime(&b, ws->event(3 * g + 1), ws->event(3 * g + 2)));
      out->ms_exact += a;
      out->ms_expand += b;
    }
    return LTSG_OK;
  };
  Cand* gbuf = nullptr;  // static generations: rows the guided pre-decision left for the exact pass
  const bool use_guide = LTSG_GUIDE && all_static && !getenv("LTSG_NO_GUIDE");
  auto launch_screen = [&](const Cand* in, int64_t n, const unsigned long long* n_in, Cand* next,
                           unsigned long long cap, unsigned long long* n_out, Cand* xbuf,
                           unsigned long long* xcnt) -> int {
    ScreenOut so{next, cap, n_in, n_out, resting, rest_cap, entries, entry_cap, cross, cross_cap, d_ctr};
    if (all_static) {
      // exact pass of the frontier (parents into xbuf, count in xcnt), then
      // the culled expansion of the parents into the next frontier
      const size_t e = 3 * n_timed++;
      LTSG_CUDA(cudaEventRecord(ws->event(e), st));
      const Cand* exact_in = in;
      const unsigned long long* exact_n = n_in;
      ScreenOut so_exact = so;
      if (use_guide) {
        // guided pre-decision: decided rows act at once, the rest are compacted into gbuf
        unsigned long long* gcnt = xcnt + (kMaxGen + 1);
        const int64_t gb = n_in ? 148LL * LTSG_GUIDE_MINB * LTSG_GUIDE_GRID : (n + kGuideThreads - 1) / kGuideThreads;
        k_guide_static<<<(int)std::max<int64_t>(1, std::min<int64_t>(gb, 148LL * LTSG_GUIDE_MINB * LTSG_GUIDE_GRID)), kGuideThreads, 0,
                         st>>>(in, n, pr.pairs, world, woff, so, reinterpret_cast<Parent*>(xbuf), xcnt, gbuf, gcnt);
        LTSG_LAUNCHED();
        exact_in = gbuf;
        exact_n = gcnt;
        so_exact.n_in = gcnt;
        so_exact.next_cap = n_in ? cap : (unsigned long long)n;  // gbuf holds at most the frontier
      }
      const int64_t blocks = exact_n ? 148LL * LTSG_STATIC_GRID : (n + 32 * kStaticWarps - 1) / (32 * kStaticWarps);
      k_screen_static<<<(int)std::max<int64_t>(1, std::min<int64_t>(blocks, 148LL * LTSG_STATIC_GRID)), 32 * kStaticWarps,
                        kStaticStageBytes, st>>>(exact_in, n, pr.pairs, pr.bodies, world, woff, so_exact,
                                                 reinterpret_cast<Parent*>(xbuf), xcnt, !use_guide);
      LTSG_LAUNCHED();
      LTSG_CUDA(cudaEventRecord(ws->event(e + 1), st));
      k_expand_filter<<<148 * LTSG_EXP_GRID, kExpThreads, 0, st>>>(reinterpret_cast<const Parent*>(xbuf), xcnt, cap, (int)fan,
                                                       world, wsph, next, cap, n_out, d_ctr);
      LTSG_LAUNCHED();
      LTSG_CUDA(cudaEventRecord(ws->event(e + 2), st));
      return LTSG_OK;
    } else if (legacy_moving) {
      const int grid = n_in ? 148 * 32 : screen_grid(n);
      k_screen<<<grid, 32 * kScreenWarps, kScreenStageBytes, st>>>(in, n, pr.pairs, pr.bodies, sc->tris, so,
                                                                   poses);
    } else {
      // cull kernel -> surviving rows (counted in xcnt) -> exact distances -> decisions
      if (cap > 0xffffffffULL) {  // rows name their candidate with a 32-bit frontier index
        set_error("moving frontier capacity %llu exceeds 2^32", cap);
        return LTSG_ECAPACITY;
      }
      const RowList rl{mrows, mrows_cap, xcnt};
      const int64_t mcap = 148LL * LTSG_MSCREEN_MINB * 64 / kMWarps;
      const int64_t mblocks = n_in ? mcap : (n + 32 * kMWarps - 1) / (32 * kMWarps);
      k_mscreen<<<(int)std::max<int64_t>(1, std::min<int64_t>(mblocks, mcap)),
                  32 * kMWarps, 0, st>>>(in, n, pr.pairs, pr.bodies, sc->tris, so, poses, rl);
      LTSG_LAUNCHED();
      const size_t e = 3 * n_timed++;
      LTSG_CUDA(cudaEventRecord(ws->event(e), st));
      k_mexact<<<148 * LTSG_MEXACT_MINB * 4, kMExactThreads, kMExactStageBytes, st>>>(in, pr.pairs, pr.bodies,
                                                                                    sc->tris, poses, rl,
                                                                                    &d_ctr->bound_rows);
      LTSG_LAUNCHED();
      LTSG_CUDA(cudaEventRecord(ws->event(e + 1), st));
      k_mdecide<<<148 * 8, 32 * kMDecideWarps, 0, st>>>(in, pr.pairs, pr.bodies, sc->tris, rl, so);
      LTSG_CUDA(cudaEventRecord(ws->event(e + 2), st));
    }
    LTSG_LAUNCHED();
    return LTSG_OK;
  };

  // static seeds: roots x roots per pair, or fine x fine (exhaustive) as
  // sphere-test tiles; both count every row and cull on the fly
  int64_t* seed_items = nullptr;
  if (all_static && sc->exhaustive && sc->n_pairs > 0) {
    int64_t* item_cnt;
    LTSG_TRY(ws_get(ws, "seed_item_cnt", (size_t)sc->n_pairs + 1, &item_cnt));
    LTSG_TRY(ws_get(ws, "seed_item_off", (size_t)sc->n_pairs + 1, &seed_items));
    k_seed_tile_count<<<grid_for(sc->n_pairs + 1, 128), 128, 0, st>>>(pr.pairs, sc->n_pairs, pr.bodies, item_cnt);
    LTSG_LAUNCHED();
    LTSG_TRY(scan_exclusive(ws, item_cnt, seed_items, sc->n_pairs + 1, st));
  }
  auto launch_static_seeds = [&](Cand* dst, size_t cap) -> int {
    if (seed_items) {
      k_seed_static_tile<<<148 * 8, kSeedTileA, 0, st>>>(pr.pairs, sc->n_pairs, pr.bodies, woff, world, wsph,
                                                         seed_items, dst, cap, d_ctr, gen_cnt);
    } else {
      k_seed_static<<<(int)std::min<int64_t>(sc->n_pairs, 148 * 16), 128, 0, st>>>(
          pr.pairs, sc->n_pairs, pr.bodies, woff, world, wsph, dst, cap, d_ctr, gen_cnt, sc->exhaustive);
    }
    LTSG_LAUNCHED();
    return LTSG_OK;
  };

  auto traverse = [&](bool async_mode, bool* overflow) -> int {
    *overflow = false;
    n_timed = 0;
    LTSG_CUDA(cudaMemsetAsync(d_ctr, 0, sizeof(Counters), st));
    LTSG_CUDA(cudaMemsetAsync(gen_cnt, 0, sizeof(unsigned long long) * (kMaxGen + 1), st));
    LTSG_CUDA(cudaMemsetAsync(x_cnt, 0, sizeof(unsigned long long) * 2 * (kMaxGen + 1), st));
    LTSG_TRY(ws_get(ws, "resting", rest_cap, &resting));
    LTSG_TRY(ws_get(ws, "entries", entry_cap, &entries));
    LTSG_TRY(ws_get(ws, "cross", cross_cap, &cross));
    out->candidates = 0;
    out->generations = 0;
    out->ms_screen = 0.0;
    if (sc->n_pairs == 0) return LTSG_OK;
    // static seeds are culled on the fly: size for the survivors (hint), grow on overflow
    const size_t hint_cap = (size_t)(1.25 * (double)ws->hint_front) + 1024;
    const size_t seed_cap = all_static ? std::min((size_t)seed_total, std::max(hint_cap, ws->hint_seed))
                                       : (size_t)seed_total;
    const size_t cap_async = std::max(hint_cap, seed_cap);
    LTSG_TRY(ws_get(ws, "front0", async_mode ? cap_async : seed_cap, &front));
    // the static seed kernel tests (and culls) the root rows: it is screen work
    t_screen.start(st);
    if (all_static) {
      LTSG_TRY(launch_static_seeds(front, seed_cap));
    } else {
      k_seed_fill<<<(int)std::min<int64_t>(sc->n_pairs, 148 * 16), 128, 0, st>>>(
          pr.pairs, sc->n_pairs, pr.bodies, sc->exhaustive, seed_off, front);
      LTSG_LAUNCHED();
      LTSG_CUDA(cudaMemcpyAsync(gen_cnt, &seed_total, sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
    }
    if (async_mode) {
      Cand* buf[2];
      buf[0] = front;
      LTSG_TRY(ws_get(ws, "front1", cap_async, &buf[1]));
      Cand* xbuf = nullptr;
      if (all_static) LTSG_TRY(ws_get(ws, "frontx", cap_async, &xbuf));
      if (all_static && use_guide) LTSG_TRY(ws_get(ws, "frontg", cap_async, &gbuf));
      if (!all_static && !legacy_moving) {
        mrows_cap = std::max(cap_async, (size_t)(1.25 * (double)ws->hint_mrows) + 1024);
        LTSG_TRY(ws_get(ws, "mrows", mrows_cap, &mrows));
      }
      // one generation more than the deepest traversal seen: a non-empty
      // frontier after the last one means the budget was short (re-run sync)
      const int n_gen = std::min(kMaxGen, std::max(1, ws->hint_gens) + 1);
      for (int g = 1; g <= n_gen; ++g)
        LTSG_TRY(launch_screen(buf[(g - 1) & 1], 0, gen_cnt + g - 1, buf[g & 1], cap_async, gen_cnt + g, xbuf,
                               x_cnt + g));
      t_screen.stop(st);
      unsigned long long hg[kMaxGen + 1];
      LTSG_CUDA(cudaMemcpyAsync(hg, gen_cnt, sizeof(hg), cudaMemcpyDeviceToHost, st));
      LTSG_TRY(read_ctr(d_ctr, &h, st));
      out->ms_screen = t_screen.ms();
      if (hg[0] > seed_cap) ws->hint_seed = std::max(ws->hint_seed, (size_t)hg[0]);
      for (int g = 0; g <= kMaxGen; ++g) {
        if (hg[g] > (g == 0 ? seed_cap : cap_async)) *overflow = true;
        if (g < kMaxGen && hg[g] > 0) {
          out->candidates += (int64_t)hg[g];
          out->generations += 1;
        }
      }
      if (hg[n_gen] > 0) *overflow = true;  // deeper than the generation budget
      if (!all_static && !legacy_moving) {
        unsigned long long hx[kMaxGen + 1];
        LTSG_CUDA(cudaMemcpyAsync(hx, x_cnt, sizeof(hx), cudaMemcpyDeviceToHost, st));
        LTSG_CUDA(cudaStreamSynchronize(st));
        for (int g = 0; g <= kMaxGen; ++g) {
          if (hx[g] > mrows_cap) *overflow = true;
          ws->hint_mrows = std::max(ws->hint_mrows, (size_t)hx[g]);
        }
      }
      if (h.resting > rest_cap || h.entries > entry_cap || h.cross > cross_cap) *overflow = true;
      return LTSG_OK;
    }
    // sync mode
    t_screen.stop(st);
    unsigned long long n_first = 0;
    LTSG_CUDA(cudaMemcpyAsync(&n_first, gen_cnt, sizeof(n_first), cudaMemcpyDeviceToHost, st));
    LTSG_TRY(read_ctr(d_ctr, &h, st));
    out->ms_screen += t_screen.ms();
    if (n_first > seed_cap) {  // more seed survivors than room: size for them and seed again
      ws->hint_seed = (size_t)n_first;
      LTSG_CUDA(cudaMemsetAsync(d_ctr, 0, sizeof(Counters), st));
      LTSG_CUDA(cudaMemsetAsync(gen_cnt, 0, sizeof(unsigned long long) * (kMaxGen + 1), st));
      LTSG_TRY(ws_get(ws, "front0", (size_t)n_first, &front));
      LTSG_TRY(launch_static_seeds(front, n_first));
      LTSG_CUDA(cudaMemcpyAsync(&n_first, gen_cnt, sizeof(n_first), cudaMemcpyDeviceToHost, st));
      LTSG_TRY(read_ctr(d_ctr, &h, st));
    }
    int64_t n_front = (int64_t)n_first;
    int fsel = 0;
    const char* fname[2] = {"front0", "front1"};
    size_t max_front = (size_t)n_front;
    while (n_front > 0) {
      // next frontier: at most n_front * fan children, usually far fewer --
      // start from the history and grow (re-running the generation) if short
      Cand* next;
      size_t next_cap = std::min((size_t)(n_front * fan),
                                 std::max((size_t)n_front * 2, (size_t)(1.25 * (double)ws->hint_front)) + 4096);
      LTSG_TRY(ws_get(ws, fname[fsel ^ 1], next_cap, &next));
      Cand* xbuf = nullptr;
      if (all_static) LTSG_TRY(ws_get(ws, "frontx", (size_t)n_front, &xbuf));
      if (all_static && use_guide) LTSG_TRY(ws_get(ws, "frontg", (size_t)n_front, &gbuf));
      if (!all_static && !legacy_moving) {
        mrows_cap = std::max(mrows_cap, std::max((size_t)n_front, ws->hint_mrows) + 1024);
        LTSG_TRY(ws_get(ws, "mrows", mrows_cap, &mrows));
      }
      Counters before = h;
      const size_t timed_before = n_timed;
      for (;;) {
        n_timed = timed_before;  // a retried generation replaces its timing
        LTSG_CUDA(cudaMemcpyAsync(d_ctr, &before, sizeof(Counters), cudaMemcpyHostToDevice, st));
        LTSG_CUDA(cudaMemsetAsync(gen_cnt + 1, 0, sizeof(unsigned long long), st));
        LTSG_CUDA(cudaMemsetAsync(x_cnt, 0, sizeof(unsigned long long), st));
        LTSG_CUDA(cudaMemsetAsync(x_cnt + (kMaxGen + 1), 0, sizeof(unsigned long long), st));
        t_screen.start(st);
        LTSG_TRY(launch_screen(front, n_front, nullptr, next, (unsigned long long)next_cap, gen_cnt + 1, xbuf,
                               x_cnt));
        t_screen.stop(st);
        LTSG_TRY(read_ctr(d_ctr, &h, st));
        out->ms_screen += t_screen.ms();
        bool grow = false;
        if (h.resting > rest_cap) {
          rest_cap = (size_t)h.resting * 2;
          LTSG_TRY(ws_get(ws, "resting", rest_cap, &resting, true));
          grow = true;
        }
        if (h.entries > entry_cap) {
          entry_cap = (size_t)h.entries * 2;
          LTSG_TRY(ws_get(ws, "entries", entry_cap, &entries, true));
          grow = true;
        }
        if (h.cross > cross_cap) {
          cross_cap = (size_t)h.cross * 2;
          LTSG_TRY(ws_get(ws, "cross", cross_cap, &cross, true));
          grow = true;
        }
        {
          unsigned long long nn_now = 0;
          LTSG_CUDA(cudaMemcpyAsync(&nn_now, gen_cnt + 1, sizeof(nn_now), cudaMemcpyDeviceToHost, st));
          LTSG_CUDA(cudaStreamSynchronize(st));
          if (nn_now > next_cap) {
            next_cap = (size_t)(1.25 * (double)nn_now) + 4096;
            LTSG_TRY(ws_get(ws, fname[fsel ^ 1], next_cap, &next));
            grow = true;
          }
        }
        if (!all_static && !legacy_moving) {
          unsigned long long nx = 0;
          LTSG_CUDA(cudaMemcpyAsync(&nx, x_cnt, sizeof(nx), cudaMemcpyDeviceToHost, st));
          LTSG_CUDA(cudaStreamSynchronize(st));
          ws->hint_mrows = std::max(ws->hint_mrows, (size_t)nx);
          if (nx > mrows_cap) {
            mrows_cap = (size_t)(1.25 * (double)nx) + 1024;
            LTSG_TRY(ws_get(ws, "mrows", mrows_cap, &mrows));
            grow = true;
          }
        }
        if (!grow) break;
      }
      unsigned long long nn = 0;
      LTSG_CUDA(cudaMemcpyAsync(&nn, gen_cnt + 1, sizeof(nn), cudaMemcpyDeviceToHost, st));
      LTSG_CUDA(cudaStreamSynchronize(st));
      if (tr.on)
        fprintf(stderr, "[ltsg trace] gen %d front %lld rows %llu window %llu sphere %llu exact %llu next %llu ms %.3f\n",
                (int)out->generations, (long long)n_front, h.rows - before.rows, h.rows_window - before.rows_window,
                h.rows_sphere - before.rows_sphere, h.screen_exact - before.screen_exact, nn, t_screen.ms());
      out->candidates += n_front;
      out->generations += 1;
      n_front = (int64_t)nn;
      max_front = std::max(max_front, (size_t)n_front);
      fsel ^= 1;
      front = next;
    }
    ws->hint_front = std::max(ws->hint_front, max_front);
    ws->hint_gens = std::max(ws->hint_gens, (int)out->generations);
    return LTSG_OK;
  };

  bool overflow = false;
  const bool try_async = ws->hint_front > 0 && !getenv("LTSG_SYNC");
  LTSG_TRY(traverse(try_async, &overflow));
  if (overflow) {
    rest_cap = std::max(rest_cap, (size_t)h.resting * 2);
    entry_cap = std::max(entry_cap, (size_t)h.entries * 2);
    cross_cap = std::max(cross_cap, (size_t)h.cross * 2);
    LTSG_TRY(traverse(false, &overflow));
  }
  if (all_static || !legacy_moving) LTSG_TRY(static_times());
  ws->hint_rest = std::max(ws->hint_rest, (size_t)h.resting);
  ws->hint_entries = std::max(ws->hint_entries, (size_t)h.entries);
  ws->hint_cross = std::max(ws->hint_cross, (size_t)h.cross);

  tr.mark("traverse");
  if (tr.on)
    fprintf(stderr, "[ltsg trace] rows %llu window %llu sphere %llu exact %llu\n", h.rows, h.rows_window,
            h.rows_sphere, h.screen_exact);
  // ---- certified zoom + bisection
  t_refine.start(st);
  const int64_t n_entries = (int64_t)h.entries;
  int64_t n_br = 0;
  if (n_entries > 0) {
    Bracket* br;
    Interval* queue;
    int64_t *spill_a, *spill_b;
    LTSG_TRY(ws_get(ws, "brackets", (size_t)n_entries, &br));
    LTSG_TRY(ws_get(ws, "zoom_spill_a", (size_t)n_entries, &spill_a));
    LTSG_TRY(ws_get(ws, "zoom_spill_b", (size_t)n_entries, &spill_b));
    // first pass: every entry with kZoomQueue intervals per queue (LTSG_ZOOM_QUEUE overrides it, to
    // exercise the spill path in tests); spilled entries re-run with 16x larger queues
    int64_t qcap = kZoomQueue;
    if (const char* q = getenv("LTSG_ZOOM_QUEUE")) qcap = std::max(1, atoi(q));
    const int64_t* sel = nullptr;
    int64_t n_zoom = n_entries;
    while (true) {
      const int zblocks = (int)std::min<int64_t>((n_zoom + kZoomWarps - 1) / kZoomWarps, 148 * 8);
      LTSG_TRY(ws_get(ws, "zoomq", (size_t)zblocks * kZoomWarps * 2 * qcap, &queue));
      LTSG_CUDA(cudaMemsetAsync(&d_ctr->overflow, 0, sizeof(unsigned long long), st));
      k_zoom<<<zblocks, 32 * kZoomWarps, 0, st>>>(entries, n_zoom, sel, pr.pairs, pr.bodies, sc->tris, queue,
                                                  (int)qcap, spill_a, br, d_ctr);
      LTSG_LAUNCHED();
      LTSG_TRY(read_ctr(d_ctr, &h, st));
      if (h.overflow == 0) break;
      n_zoom = (int64_t)h.overflow;
      qcap *= 16;
      if (qcap > ((int64_t)1 << 26)) {
        set_error("zoom: %lld entries need more than %lld pending intervals", (long long)n_zoom, (long long)(qcap / 16));
        return LTSG_ECAPACITY;
      }
      std::swap(spill_a, spill_b);  // the spilled list becomes the selection; the next pass spills into the other
      sel = spill_b;
    }
    n_br = (int64_t)h.brackets;
    if (n_br > 0) {
      const size_t need = (size_t)(h.cross + n_br);
      if (need > cross_cap) {
        cross_cap = need;
        LTSG_TRY(ws_get(ws, "cross", cross_cap, &cross, true));
      }
      k_bisect<<<grid_for(n_br, 64), 64, 0, st>>>(br, n_br, pr.pairs, pr.bodies, sc->tris, cross, h.cross,
                                                 tau_min);
      LTSG_LAUNCHED();
    }
  }
  const int64_t n_cross = (int64_t)h.cross + n_br;
  t_refine.stop(st);
  tr.mark("refine");
  t_contacts.start(st);
  k_finalize<<<grid_for(np, 128), 128, 0, st>>>(tau_min, sc->problem_dt, np, sc->widen, out->dt,
                                                out->first_contact, out->collision);
  LTSG_LAUNCHED();

  // ---- records
  const int64_t n_rest = (int64_t)h.resting;
  const int64_t n_cand_rec = n_rest + n_cross;
  Record* recs;
  LTSG_TRY(ws_get(ws, "records", (size_t)n_cand_rec, &recs));
  if (n_cand_rec > 0) {
    k_collect<<<grid_for(n_cand_rec, 128), 128, 0, st>>>(resting, n_rest, cross, n_cross, pr.pairs, out->dt,
                                                        recs, d_ctr);
    LTSG_LAUNCHED();
  }
  LTSG_TRY(read_ctr(d_ctr, &h, st));
  tr.mark("collect");
  const int64_t n_rec = (int64_t)h.records;
  out->rows_screen = (int64_t)h.rows;
  out->rows_zoom = (int64_t)h.zoom_rows;
  out->rows_bisect = n_br * kBisectIters;
  out->rows_executed = (int64_t)(h.screen_exact + h.zoom_exec) + n_br * kBisectIters;
  out->rows_screen_exact = (int64_t)(h.screen_exact - h.bound_rows);
  out->rows_bound = (int64_t)h.bound_rows;
  out->n_raw = n_rec;

  int32_t* prob_count;
  int64_t *prob_count64;
  LTSG_TRY(ws_get(ws, "prob_count", (size_t)np + 1, &prob_count));
  LTSG_TRY(ws_get(ws, "prob_count64", (size_t)np + 1, &prob_count64));
  LTSG_CUDA(cudaMemsetAsync(prob_count, 0, sizeof(int32_t) * (np + 1), st));
  if (n_rec == 0) {
    LTSG_CUDA(cudaMemsetAsync(out->fused_offset, 0, sizeof(int64_t) * (np + 1), st));
    out->n_fused = 0;
    t_contacts.stop(st);
    LTSG_CUDA(cudaStreamSynchronize(st));
    out->ms_refine = t_refine.ms();
    out->ms_contacts = t_contacts.ms();
    return LTSG_OK;
  }
  if (n_rec > out->capacity) {
    set_error("contact capacity %lld < %lld raw contacts", (long long)out->capacity, (long long)n_rec);
    out->n_fused = n_rec;
    return LTSG_ECAPACITY;
  }

  // ---- contact records (raw, record order)
  Soa ro;
  unsigned long long* key;
  LTSG_TRY(ws_get(ws, "r_problem", n_rec, &ro.problem));
  LTSG_TRY(ws_get(ws, "r_body_a", n_rec, &ro.body_a));
  LTSG_TRY(ws_get(ws, "r_body_b", n_rec, &ro.body_b));
  LTSG_TRY(ws_get(ws, "r_pos", 3 * n_rec, &ro.position));
  LTSG_TRY(ws_get(ws, "r_nrm", 3 * n_rec, &ro.normal));
  LTSG_TRY(ws_get(ws, "r_depth", n_rec, &ro.depth));
  LTSG_TRY(ws_get(ws, "r_t", n_rec, &ro.t));
  LTSG_TRY(ws_get(ws, "r_tri_a", n_rec, &ro.tri_a));
  LTSG_TRY(ws_get(ws, "r_tri_b", n_rec, &ro.tri_b));
  LTSG_TRY(ws_get(ws, "r_thr", n_rec, &ro.threshold));
  LTSG_TRY(ws_get(ws, "r_key", n_rec, &key));
  k_contacts<<<grid_for(n_rec, 64), 64, 0, st>>>(recs, n_rec, pr.pairs, pr.bodies, sc->tris, sc->tri_orig,
                                                 sc->problem_tbase, ro, key);
  LTSG_LAUNCHED();
  tr.mark("contacts");
  LTSG_TRY(fuse_stage(ws, st, ro, key, n_rec, np, prob_count, prob_count64, out));
  tr.mark("fuse");
  t_contacts.stop(st);
  out->ms_refine = t_refine.ms();
  out->ms_contacts = t_contacts.ms();
  return LTSG_OK;
}

// Group raw records by (problem, body pair), fuse each group
// (filter_contacts), write raw (canonical order) and fused outputs.
static int fuse_stage(ltsg_workspace* ws, cudaStream_t st, Soa ro, unsigned long long* key, int64_t n_rec,
                      int np, int32_t* prob_count, int64_t* prob_count64, ltsg_result* out) {
  // group by (problem, body pair): radix sort of the group key
  int64_t *idx_in, *idx, *head, *head_scan, *g_off, *g_fused, *g_dst;
  unsigned long long* keys_sorted;
  int32_t* parent;
  LTSG_TRY(ws_get(ws, "idx_in", n_rec, &idx_in));
  LTSG_TRY(ws_get(ws, "idx", n_rec, &idx));
  LTSG_TRY(ws_get(ws, "keys_sorted", n_rec, &keys_sorted));
  LTSG_TRY(ws_get(ws, "head", n_rec + 1, &head));
  LTSG_TRY(ws_get(ws, "head_scan", n_rec + 1, &head_scan));
  LTSG_TRY(ws_get(ws, "parent", n_rec, &parent));
  k_iota<<<grid_for(n_rec, 256), 256, 0, st>>>(idx_in, n_rec);
  LTSG_LAUNCHED();
  {
    size_t tmp = 0;
    // keys are (problem << 32) | rank with problem < np: the bits above
    // 32 + bit_width(np) are zero, so fewer radix passes sort them
    int end_bit = 32;
    while (end_bit < 64 && ((unsigned long long)np >> (end_bit - 32)) != 0) ++end_bit;
    LTSG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, keys_sorted, idx_in, idx, n_rec, 0, end_bit, st));
    void* t;
    LTSG_TRY(ws->get("cub_tmp", tmp, &t));
    LTSG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key, keys_sorted, idx_in, idx, n_rec, 0, end_bit, st));
  }
  k_heads<<<grid_for(n_rec + 1, 256), 256, 0, st>>>(keys_sorted, n_rec, head);
  LTSG_LAUNCHED();
  LTSG_TRY(scan_exclusive(ws, head, head_scan, n_rec + 1, st));
  int64_t n_groups = 0;
  LTSG_CUDA(cudaMemcpyAsync(&n_groups, head_scan + n_rec, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  LTSG_TRY(ws_get(ws, "g_off", (size_t)n_groups + 1, &g_off));
  LTSG_TRY(ws_get(ws, "g_fused", (size_t)n_groups + 1, &g_fused));
  LTSG_TRY(ws_get(ws, "g_dst", (size_t)n_groups + 1, &g_dst));
  k_group_table<<<grid_for(n_rec, 256), 256, 0, st>>>(head, head_scan, n_rec, g_off);
  LTSG_LAUNCHED();

  Soa fs;  // fused, group-slotted
  LTSG_TRY(ws_get(ws, "f_problem", n_rec, &fs.problem));
  LTSG_TRY(ws_get(ws, "f_body_a", n_rec, &fs.body_a));
  LTSG_TRY(ws_get(ws, "f_body_b", n_rec, &fs.body_b));
  LTSG_TRY(ws_get(ws, "f_pos", 3 * n_rec, &fs.position));
  LTSG_TRY(ws_get(ws, "f_nrm", 3 * n_rec, &fs.normal));
  LTSG_TRY(ws_get(ws, "f_depth", n_rec, &fs.depth));
  LTSG_TRY(ws_get(ws, "f_t", n_rec, &fs.t));
  LTSG_TRY(ws_get(ws, "f_tri_a", n_rec, &fs.tri_a));
  LTSG_TRY(ws_get(ws, "f_tri_b", n_rec, &fs.tri_b));
  LTSG_TRY(ws_get(ws, "f_thr", n_rec, &fs.threshold));
  int32_t *big_list, *big_count;
  LTSG_TRY(ws_get(ws, "big_list", (size_t)n_groups, &big_list));
  LTSG_TRY(ws_get(ws, "big_count", 1, &big_count));
  LTSG_CUDA(cudaMemsetAsync(big_count, 0, sizeof(int32_t), st));
  k_fuse_block<<<(int)std::min<int64_t>(n_groups, 148 * 8), kFuseThreads, 0, st>>>(
      ro, idx, g_off, n_groups, n_rec, fs, g_fused, prob_count, big_list, big_count);
  LTSG_LAUNCHED();
  int32_t n_big = 0;
  LTSG_CUDA(cudaMemcpyAsync(&n_big, big_count, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  if (n_big > 0) {
    std::vector<int32_t> hb(n_big);
    std::vector<int64_t> hoff(n_groups + 1);
    LTSG_CUDA(cudaMemcpyAsync(hb.data(), big_list, sizeof(int32_t) * n_big, cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaMemcpyAsync(hoff.data(), g_off, sizeof(int64_t) * n_groups, cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaStreamSynchronize(st));
    hoff[n_groups] = n_rec;
    std::vector<int64_t> aoff(n_big + 1, 0);
    for (int b = 0; b < n_big; ++b) {
      const int64_t n = hoff[hb[b] + 1] - hoff[hb[b]];
      aoff[b + 1] = aoff[b] + n * ((n + 31) / 32);
    }
    int64_t* d_aoff;
    uint32_t* adj;
    FuseKey* keys;
    int64_t* gi;
    double *pos, *thr;
    int32_t* slot;
    LTSG_TRY(ws_get(ws, "fl_aoff", (size_t)n_big + 1, &d_aoff));
    LTSG_TRY(ws_get(ws, "fl_adj", (size_t)aoff[n_big], &adj));
    LTSG_TRY(ws_get(ws, "fl_keys", (size_t)n_rec, &keys));
    LTSG_TRY(ws_get(ws, "fl_gi", (size_t)n_rec, &gi));
    LTSG_TRY(ws_get(ws, "fl_pos", (size_t)n_rec * 3, &pos));
    LTSG_TRY(ws_get(ws, "fl_thr", (size_t)n_rec, &thr));
    LTSG_TRY(ws_get(ws, "fl_slot", (size_t)n_rec, &slot));
    LTSG_CUDA(cudaMemcpyAsync(d_aoff, aoff.data(), sizeof(int64_t) * (n_big + 1), cudaMemcpyHostToDevice, st));
    k_fuse_large<<<n_big, kFuseLargeThreads, 0, st>>>(ro, idx, g_off, n_groups, n_rec, fs, g_fused, prob_count,
                                                      big_list, d_aoff, keys, gi, pos, thr, parent, slot, adj);
    LTSG_LAUNCHED();
  }

  // raw output in canonical order (group, then fusion key)
  if (out->raw_t) {
    Soa rr{out->raw_problem, out->raw_body_a, out->raw_body_b, out->raw_position, out->raw_normal,
           out->raw_depth, out->raw_t, out->raw_tri_a, out->raw_tri_b, out->raw_threshold};
    k_gather<<<grid_for(n_rec, 128), 128, 0, st>>>(ro, idx, n_rec, rr);
    LTSG_LAUNCHED();
  }
  // dense fused output
  LTSG_CUDA(cudaMemsetAsync(g_fused + n_groups, 0, sizeof(int64_t), st));
  LTSG_TRY(scan_exclusive(ws, g_fused, g_dst, n_groups + 1, st));
  Soa fo{out->problem, out->body_a, out->body_b, out->position, out->normal, out->depth, out->t,
         out->tri_a, out->tri_b, out->threshold};
  k_compact<<<(int)std::min<int64_t>(n_groups, 148 * 16), 64, 0, st>>>(fs, g_off, g_fused, g_dst, n_groups, fo);
  LTSG_LAUNCHED();
  k_widen<<<grid_for(np + 1, 256), 256, 0, st>>>(prob_count, prob_count64, np + 1);
  LTSG_LAUNCHED();
  LTSG_TRY(scan_exclusive(ws, prob_count64, out->fused_offset, np + 1, st));
  LTSG_CUDA(cudaMemcpyAsync(&out->n_fused, g_dst + n_groups, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  return LTSG_OK;
}

static int build_world(const ltsg_scene* sc, const Prepared& pr, ltsg_workspace* ws, cudaStream_t st,
                       double** world, int64_t** woff, int64_t* n_world, int* launches) {
  int64_t* wcnt;
  LTSG_TRY(ws_get(ws, "world_cnt", (size_t)sc->n_bodies + 1, &wcnt));
  LTSG_TRY(ws_get(ws, "world_off", (size_t)sc->n_bodies + 1, woff));
  k_world_count<<<grid_for(sc->n_bodies + 1, 128), 128, 0, st>>>(pr.bodies, sc->n_bodies, wcnt);
  LTSG_CHECK_LAUNCH();
  LTSG_TRY(scan_exclusive(ws, wcnt, *woff, sc->n_bodies + 1, st));
  LTSG_CUDA(cudaMemcpyAsync(n_world, *woff + sc->n_bodies, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  if (*n_world >= (int64_t)1 << 31) {
    *world = nullptr;
    return LTSG_OK;
  }
  LTSG_TRY(ws_get(ws, "world", (size_t)std::max<int64_t>(*n_world, 1) * (kWorld + kSph), world));
  k_world_fill<<<(int)std::max<int64_t>(1, std::min<int64_t>((*n_world + 127) / 128, 148 * 16)), 128, 0, st>>>(
      pr.bodies, sc->n_bodies, *woff,
                                                                              sc->tris, *world,
                                                                              *world + (size_t)std::max<int64_t>(*n_world, 1) * kWorld);
  LTSG_CHECK_LAUNCH();
  *launches += 2;
  return LTSG_OK;
}

static int run_allpairs(const ltsg_scene* sc, int64_t* rows, int64_t* hits, double* ms, double* out_dist,
                        ltsg_workspace* ws, cudaStream_t st) {
  LTSG_TRY(validate(sc));
  LTSG_TRY(configure_kernels());
  Prepared pr{};
  LTSG_TRY(prepare(sc, ws, st, &pr));
  unsigned long long* d_hits;
  LTSG_TRY(ws_get(ws, "hits", 1, &d_hits));
  LTSG_CUDA(cudaMemsetAsync(d_hits, 0, sizeof(unsigned long long), st));
  *rows = 0;
  *ms = 0.0;
  if (sc->n_pairs > 0 && sc->n_bodies > 0) {
    double* world;
    int64_t* woff;
    int64_t n_world = 0;
    int launches = 0;
    LTSG_TRY(build_world(sc, pr, ws, st, &world, &woff, &n_world, &launches));
    if (!world) {
      set_error("ltsg_exhaustive_rows: scene too large for the world cache");
      return LTSG_ECAPACITY;
    }
    // rows = sum over pairs of fine sizes product (host-side from the level tables)
    std::vector<int64_t> lev((size_t)sc->n_bodies * 18);
    std::vector<int32_t> pb((size_t)sc->n_pairs * 2);
    LTSG_CUDA(cudaMemcpyAsync(lev.data(), sc->body_levels, sizeof(int64_t) * lev.size(), cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaMemcpyAsync(pb.data(), sc->pair_body, sizeof(int32_t) * pb.size(), cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaStreamSynchronize(st));
    for (int64_t k = 0; k < sc->n_pairs; ++k) *rows += lev[(size_t)pb[2 * k] * 18 + 10] * lev[(size_t)pb[2 * k + 1] * 18 + 10];
    // per-pair prefixes of tile items and of rows (row-major na x nb per pair)
    std::vector<int64_t> items((size_t)sc->n_pairs + 1, 0), rowv((size_t)sc->n_pairs + 1, 0);
    for (int64_t k = 0; k < sc->n_pairs; ++k) {
      const int64_t na = lev[(size_t)pb[2 * k] * 18 + 10], nb = lev[(size_t)pb[2 * k + 1] * 18 + 10];
      items[k + 1] = items[k] + ((na + kTileA - 1) / kTileA) * ((nb + kTileB - 1) / kTileB);
      rowv[k + 1] = rowv[k] + na * nb;
    }
    int64_t *d_items, *d_rows;
    LTSG_TRY(ws_get(ws, "tile_items", items.size(), &d_items));
    LTSG_TRY(ws_get(ws, "tile_rows", rowv.size(), &d_rows));
    LTSG_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(int64_t) * items.size(), cudaMemcpyHostToDevice, st));
    LTSG_CUDA(cudaMemcpyAsync(d_rows, rowv.data(), sizeof(int64_t) * rowv.size(), cudaMemcpyHostToDevice, st));
    Timer t;
    t.start(st);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(items.back(), 148LL * LTSG_TILE_MINB * 8));
    k_allpairs_tile<<<grid, kTileA, kTileSmemBytes, st>>>(pr.pairs, sc->n_pairs, pr.bodies, world, woff, d_items,
                                                          d_rows, d_hits, out_dist);
    t.stop(st);
    LTSG_CHECK_LAUNCH();
    *ms = t.ms();
  }
  unsigned long long h = 0;
  LTSG_CUDA(cudaMemcpyAsync(&h, d_hits, sizeof(h), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  *hits = (int64_t)h;
  return LTSG_OK;
}

}  // namespace ltsg

extern "C" int ltsg_search(const ltsg_scene* scene, ltsg_result* out, ltsg_workspace* ws, void* stream) {
  if (!scene || !out || !ws) {
    ltsg::set_error("ltsg_search: null argument");
    return LTSG_EINVAL;
  }
  return ltsg::run_search(scene, out, ws, (cudaStream_t)stream);
}

extern "C" int ltsg_fuse_contacts(ltsg_result* io, int64_t n_raw, const uint64_t* group_key,
                                  ltsg_workspace* ws, void* stream) {
  using namespace ltsg;
  if (!io || !ws || n_raw < 0 || (n_raw > 0 && (!group_key || !io->raw_t || !io->raw_problem))) {
    set_error("ltsg_fuse_contacts: invalid arguments");
    return LTSG_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // n_problems = 1 + max problem id, passed through io->n_raw on entry
  const int np = (int)io->n_raw;
  if (np < 1) {
    set_error("ltsg_fuse_contacts: io->n_raw must carry the problem count (>= 1)");
    return LTSG_EINVAL;
  }
  io->n_fused = 0;
  if (n_raw > io->capacity) {
    set_error("ltsg_fuse_contacts: capacity %lld < %lld", (long long)io->capacity, (long long)n_raw);
    return LTSG_ECAPACITY;
  }
  int32_t* prob_count;
  int64_t* prob_count64;
  LTSG_TRY(ws_get(ws, "prob_count", (size_t)np + 1, &prob_count));
  LTSG_TRY(ws_get(ws, "prob_count64", (size_t)np + 1, &prob_count64));
  LTSG_CUDA(cudaMemsetAsync(prob_count, 0, sizeof(int32_t) * (np + 1), st));
  io->n_raw = n_raw;
  if (n_raw == 0) {
    LTSG_CUDA(cudaMemsetAsync(io->fused_offset, 0, sizeof(int64_t) * (np + 1), st));
    LTSG_CUDA(cudaStreamSynchronize(st));
    return LTSG_OK;
  }
  Soa ro{io->raw_problem, io->raw_body_a, io->raw_body_b, io->raw_position, io->raw_normal,
         io->raw_depth, io->raw_t, io->raw_tri_a, io->raw_tri_b, io->raw_threshold};
  unsigned long long* key;
  LTSG_TRY(ws_get(ws, "r_key", (size_t)n_raw, &key));
  LTSG_CUDA(cudaMemcpyAsync(key, group_key, sizeof(uint64_t) * n_raw, cudaMemcpyDeviceToDevice, st));
  // the raw arrays are inputs here: do not overwrite them with the canonical order
  double* saved_raw_t = io->raw_t;
  io->raw_t = nullptr;
  const int rc = fuse_stage(ws, st, ro, key, n_raw, np, prob_count, prob_count64, io);
  io->raw_t = saved_raw_t;
  return rc;
}

extern "C" int ltsg_exhaustive_rows(const ltsg_scene* scene, int64_t* rows, int64_t* hits, double* ms,
                                    ltsg_workspace* ws, void* stream) {
  if (!scene || !rows || !hits || !ms || !ws) {
    ltsg::set_error("ltsg_exhaustive_rows: null argument");
    return LTSG_EINVAL;
  }
  return ltsg::run_allpairs(scene, rows, hits, ms, nullptr, ws, (cudaStream_t)stream);
}

extern "C" int ltsg_exhaustive_distances(const ltsg_scene* scene, double* out_dist, int64_t* rows,
                                         ltsg_workspace* ws, void* stream) {
  if (!scene || !out_dist || !rows || !ws) {
    ltsg::set_error("ltsg_exhaustive_distances: null argument");
    return LTSG_EINVAL;
  }
  int64_t hits = 0;
  double ms = 0.0;
  return ltsg::run_allpairs(scene, rows, &hits, &ms, out_dist, ws, (cudaStream_t)stream);
}
