// Space-time broad phase on sm_100a: the collision graph that feeds the
// narrow phase (ltsdem.broadphase.build_collision_graph, broadphase.py:198-252).
//
// Pipeline (one call, one stream):
//   k_bp_traj   one thread per body: step bound (particle_dt, :46-50), the
//               piecewise-linear sphere-centre trajectory (_Trajectory.of_particle
//               / of_static, :83-99; extrapolate_free_flight state.py:89-99;
//               sphere_center_at body.py:36-37) and its time-collapsed box
//               (_Trajectory.box, :115-118).  The sort key is the box's lo.x.
//   cub radix sort of the bodies by lo.x.
//   k_bp_sweep  sort-and-sweep over tiles of 128 sorted boxes staged in shared
//               memory: Check 1 (check_spacetime_aabb, :121-125) on every pair
//               whose x-extents overlap.  The reference's uniform hash
//               (_hash_candidates, :161-195) is "an acceleration only, never a
//               filter" -- every box-overlapping pair shares a cell -- so any
//               complete enumeration of box-overlapping pairs gives the same
//               graph; the sweep is the GPU-shaped one.  Two statics are never
//               paired (:228-229).
//   k_bp_tube   one thread per surviving pair: the pair window (pair_window
//               :53-56, or (old.t, t_cur + dt) against a static, :240-243) and
//               Check 2 (check_spacetime_tube / _min_distance_over_window,
//               :128-158) with the reference's knots and rounding; survivors
//               become edges (two particles) or static links.
//   cub radix sorts put edges in the reference's dict order (sorted
//   (index_a, index_b)) and static links in (particle, static id) order.
//
// Rounding: numpy elementwise operations are separately rounded (this file
// is compiled with -fmad=false and uses explicit __d*_rn); 1-D `@` and
// np.linalg.norm are OpenBLAS ddot FMA chains (dot_blas, geom.cuh).  So the
// graph is bit-identical to the reference's.  The one transcendental on the
// path, quaternions.advance's sin/cos for the extrapolated rotation, only
// matters for a sphere centre off the body origin (make_particle pins it at
// the origin, body.py:73-76), where rotate(q, 0) is exactly 0.
#include "common.cuh"
#include "geom.cuh"
#include "quat.cuh"

#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>

namespace ltsg {
namespace bp {

constexpr int kRec = 28;  // particle record, see ltsgpu.h (ltsg_broad_input)
constexpr int kTile = 128;

struct Traj {
  double t[3];
  double c[9];
  double r;
  int32_t nt;
  int32_t pad;
};

struct Cand {
  int32_t a, b;  // body indices, a < b, a a particle
};

__device__ __forceinline__ V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }

// ---------------------------------------------------------------- trajectories
// _Trajectory.at (:101-113)
__device__ __forceinline__ V3 traj_at(const Traj& tr, double t) {
  const V3 c0{tr.c[0], tr.c[1], tr.c[2]};
  if (tr.nt == 1) return c0;
  const V3 c1{tr.c[3], tr.c[4], tr.c[5]};
  const V3 c2{tr.c[6], tr.c[7], tr.c[8]};
  if (tr.t[0] > t) t = tr.t[0];  // Python max(t, times[0])
  if (tr.t[2] < t) t = tr.t[2];  // Python min(., times[-1])
  V3 a = c1, b = c2;
  double ta = tr.t[1], tb = tr.t[2];
  if (t <= tr.t[1]) {
    a = c0;
    b = c1;
    ta = tr.t[0];
    tb = tr.t[1];
  }
  const double span = sub(tb, ta);
  if (span == 0.0) return b;
  const double u = dv(sub(t, ta), span);
  return scale(a, sub(1.0, u)) + scale(b, u);
}

// _min_distance_over_window (:128-151)
__device__ double min_distance(const Traj& t1, const Traj& t2, double w0, double w1) {
  if (w1 < w0) return CUDART_INF;
  // the knot set {w0, w1} u {trajectory times strictly inside}, sorted
  double k[8];
  int nk = 0;
  auto insert = [&](double v) {
    for (int i = 0; i < nk; ++i)
      if (k[i] == v) return;  // set semantics: an equal value is already there
    int i = nk++;
    while (i > 0 && k[i - 1] > v) {
      k[i] = k[i - 1];
      --i;
    }
    k[i] = v;
  };
  insert(w0);
  insert(w1);
  for (int i = 0; i < t1.nt; ++i)
    if (w0 < t1.t[i] && t1.t[i] < w1) insert(t1.t[i]);
  for (int i = 0; i < t2.nt; ++i)
    if (w0 < t2.t[i] && t2.t[i] < w1) insert(t2.t[i]);
  double best = CUDART_INF;
  V3 d0 = traj_at(t1, k[0]) - traj_at(t2, k[0]);
  if (nk == 1) return norm_blas(d0);
  for (int i = 1; i < nk; ++i) {
    const V3 d1 = traj_at(t1, k[i]) - traj_at(t2, k[i]);
    const V3 dd = d1 - d0;
    const double denom = dot_blas(dd, dd);
    double s = 0.0;
    if (denom != 0.0) {
      s = dv(-dot_blas(d0, dd), denom);
      s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);  // np.clip (NaN passes)
    }
    const double d = norm_blas(d0 + scale(dd, s));
    if (d < best) best = d;  // Python min(best, d)
    d0 = d1;
  }
  return best;
}

__device__ __forceinline__ uint64_t order_key(double x) {  // ascending doubles -> ascending uint64
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_bp_traj(const double* __restrict__ rec, const double* __restrict__ srec, int n_p, int n_s,
                          double dt_max, double growth, Traj* __restrict__ traj, double* __restrict__ box,
                          double* __restrict__ dts, uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_p + n_s) return;
  Traj tr{};
  if (i < n_p) {
    const double* r = rec + (size_t)i * kRec;
    const double old_t = r[7], cur_t = r[15];
    const double last = sub(cur_t, old_t);  // particle_dt (:46-50)
    double dt = dt_max;
    if (last != 0.0) {
      const double g = mul(growth, last);
      dt = dt_max < g ? dt_max : g;
    }
    dts[i] = dt;
    const V3 centre = ld3(r + 22);
    const V3 cur_pos = ld3(r + 8);
    const V3 ext_pos = cur_pos + scale(ld3(r + 16), dt);  // extrapolate_free_flight (state.py:94)
    V3 c_old = ld3(r), c_cur = cur_pos, c_ext = ext_pos;
    if (centre.x != 0.0 || centre.y != 0.0 || centre.z != 0.0) {
      // sphere_center_at = position + rotate(rotation, centre); for a centre at
      // the origin rotate() is exactly zero and is skipped
      double q_ext[4];
      advance(r + 11, ld3(r + 19), dt, q_ext);
      c_old = c_old + rotate(r + 3, centre);
      c_cur = c_cur + rotate(r + 11, centre);
      c_ext = c_ext + rotate(q_ext, centre);
    }
    tr.t[0] = old_t;
    tr.t[1] = cur_t;
    tr.t[2] = add(cur_t, dt);
    tr.c[0] = c_old.x; tr.c[1] = c_old.y; tr.c[2] = c_old.z;
    tr.c[3] = c_cur.x; tr.c[4] = c_cur.y; tr.c[5] = c_cur.z;
    tr.c[6] = c_ext.x; tr.c[7] = c_ext.y; tr.c[8] = c_ext.z;
    tr.r = r[25];
    tr.nt = 3;
  } else {
    const double* s = srec + (size_t)(i - n_p) * 4;
    tr.c[0] = s[0]; tr.c[1] = s[1]; tr.c[2] = s[2];
    tr.r = s[3];
    tr.nt = 1;
  }
  traj[i] = tr;
  double lo[3], hi[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double mn = tr.c[d], mx = tr.c[d];
    for (int k = 1; k < tr.nt; ++k) {
      mn = fmin(mn, tr.c[3 * k + d]);
      mx = fmax(mx, tr.c[3 * k + d]);
    }
    lo[d] = sub(mn, tr.r);
    hi[d] = add(mx, tr.r);
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    box[(size_t)i * 6 + d] = lo[d];
    box[(size_t)i * 6 + 3 + d] = hi[d];
  }
  key[i] = order_key(lo[0]);
  idx[i] = i;
}

// boxes in lo.x order, structure-of-arrays (lo x y z, hi x y z, body)
__global__ void k_bp_gather(const double* __restrict__ box, const int32_t* __restrict__ order, int n,
                            double* __restrict__ sbox, int32_t* __restrict__ sbody) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = order[i];
#pragma unroll
  for (int d = 0; d < 6; ++d) sbox[(size_t)d * n + i] = box[(size_t)b * 6 + d];
  sbody[i] = b;
}

// Sort-and-sweep Check 1.  Block (ti, chunk): the 128 sorted boxes of tile ti
// against tiles ti + chunk*tpc ... (+tpc); a tile whose first lo.x exceeds the
// largest hi.x of tile ti ends the sweep for the whole block, a box past a
// lane's own hi.x ends it for the lane (boxes are in lo.x order).
__global__ void __launch_bounds__(kTile) k_bp_sweep(const double* __restrict__ sbox, const int32_t* __restrict__ sbody,
                                                    int n, int n_p, int tpc, Cand* __restrict__ cand,
                                                    unsigned long long* __restrict__ n_cand,
                                                    unsigned long long cap) {
  __shared__ double s_b[6][kTile];
  __shared__ int32_t s_id[kTile];
  __shared__ double s_red[kTile / 32];
  const int n_tiles = (n + kTile - 1) / kTile;
  const int ti = blockIdx.x;
  const int tj0 = ti + blockIdx.y * tpc;
  if (tj0 >= n_tiles) return;
  const int tj1 = min(n_tiles, tj0 + tpc);
  const int i = ti * kTile + threadIdx.x;
  const bool valid = i < n;
  double me[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) me[d] = valid ? sbox[(size_t)d * n + i] : -CUDART_INF;
  const int my_body = valid ? sbody[i] : -1;
  double m = me[3];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
  __syncthreads();
  double tile_hi = s_red[0];
#pragma unroll
  for (int w = 1; w < kTile / 32; ++w) tile_hi = fmax(tile_hi, s_red[w]);
  bool done = !valid;
  for (int tj = tj0; tj < tj1; ++tj) {
    if (sbox[tj * kTile] > tile_hi) break;  // block-uniform
    __syncthreads();
    const int j = tj * kTile + threadIdx.x;
    if (j < n) {
#pragma unroll
      for (int d = 0; d < 6; ++d) s_b[d][threadIdx.x] = sbox[(size_t)d * n + j];
      s_id[threadIdx.x] = sbody[j];
    }
    __syncthreads();
    if (!done) {
      const int kmax = min(kTile, n - tj * kTile);
      for (int k = (tj == ti ? threadIdx.x + 1 : 0); k < kmax; ++k) {
        if (s_b[0][k] > me[3]) {  // this and every later box starts past my hi.x
          done = true;
          break;
        }
        // check_spacetime_aabb: lo1 <= hi2 and lo2 <= hi1 on every axis
        const bool ov = me[0] <= s_b[3][k] && me[1] <= s_b[4][k] && me[2] <= s_b[5][k] &&
                        s_b[0][k] <= me[3] && s_b[1][k] <= me[4] && s_b[2][k] <= me[5];
        if (!ov) continue;
        const int ob = s_id[k];
        const int a = min(my_body, ob), b = max(my_body, ob);
        if (a >= n_p) continue;  // two statics never meet
        const unsigned long long slot = atomicAdd(n_cand, 1ull);
        if (slot < cap) cand[slot] = Cand{a, b};
      }
    }
  }
}

// Check 2 per candidate; survivors become edges or static links (unordered)
__global__ void k_bp_tube(const Cand* __restrict__ cand, const unsigned long long* __restrict__ n_cand_p,
                          const Traj* __restrict__ traj, const double* __restrict__ rec,
                          const double* __restrict__ dts, int n_p, int n_s, uint64_t* __restrict__ ekey,
                          double* __restrict__ ewin, int32_t* __restrict__ eperm,
                          unsigned long long* __restrict__ n_edge,
                          uint64_t* __restrict__ lkey, unsigned long long* __restrict__ n_link) {
  const int64_t n_cand = (int64_t)*n_cand_p;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cand; c += (int64_t)gridDim.x * blockDim.x) {
    const Cand p = cand[c];
    const bool dyn = p.b < n_p;
    double w0, w1;
    if (dyn) {  // pair_window (:53-56)
      const double t1 = rec[(size_t)p.a * kRec + 15], t2 = rec[(size_t)p.b * kRec + 15];
      const double d1 = dts[p.a], d2 = dts[p.b];
      const double start = t2 < t1 ? t2 : t1;
      w0 = start;
      w1 = add(start, d2 < d1 ? d2 : d1);
    } else {  // (old.t, t_cur + dt) against a static (:240-243)
      w0 = rec[(size_t)p.a * kRec + 7];
      w1 = add(rec[(size_t)p.a * kRec + 15], dts[p.a]);
    }
    const Traj ta = traj[p.a], tb = traj[p.b];
    const double best = min_distance(ta, tb, w0, w1);
    if (!(best <= add(ta.r, tb.r))) continue;  // check_spacetime_tube (:154-158)
    if (dyn) {
      const unsigned long long s = atomicAdd(n_edge, 1ull);
      ekey[s] = (uint64_t)p.a * (uint64_t)n_p + (uint64_t)p.b;
      eperm[s] = (int32_t)s;
      ewin[2 * s] = w0;
      ewin[2 * s + 1] = w1;
    } else {
      const unsigned long long s = atomicAdd(n_link, 1ull);
      lkey[s] = (uint64_t)p.a * (uint64_t)n_s + (uint64_t)(p.b - n_p);
    }
  }
}

__global__ void k_bp_emit(const uint64_t* __restrict__ ekey, const int32_t* __restrict__ eperm,
                          const double* __restrict__ ewin, int64_t n_e, int n_p, int32_t* __restrict__ edge,
                          double* __restrict__ window, const uint64_t* __restrict__ lkey, int64_t n_l, int n_s,
                          int32_t* __restrict__ link) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n_e) {
    const uint64_t k = ekey[i];
    edge[2 * i] = (int32_t)(k / (uint64_t)n_p);
    edge[2 * i + 1] = (int32_t)(k % (uint64_t)n_p);
    const int32_t s = eperm[i];
    window[2 * i] = ewin[2 * s];
    window[2 * i + 1] = ewin[2 * s + 1];
  }
  if (i < n_l) {
    const uint64_t k = lkey[i];
    link[2 * i] = (int32_t)(k / (uint64_t)n_s);
    link[2 * i + 1] = (int32_t)(k % (uint64_t)n_s);
  }
}

// ltsg_tube_rows: Check 2 on explicit trajectory rows
__global__ void k_bp_tube_rows(const double* __restrict__ t1, const double* __restrict__ c1,
                               const double* __restrict__ r1, const int32_t* __restrict__ nt1,
                               const double* __restrict__ t2, const double* __restrict__ c2,
                               const double* __restrict__ r2, const int32_t* __restrict__ nt2,
                               const double* __restrict__ win, int64_t n, double* __restrict__ dist,
                               int32_t* __restrict__ hit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Traj a{}, b{};
    for (int k = 0; k < 3; ++k) {
      a.t[k] = t1[3 * i + k];
      b.t[k] = t2[3 * i + k];
    }
    for (int k = 0; k < 9; ++k) {
      a.c[k] = c1[9 * i + k];
      b.c[k] = c2[9 * i + k];
    }
    a.r = r1[i];
    b.r = r2[i];
    a.nt = nt1[i];
    b.nt = nt2[i];
    const double d = min_distance(a, b, win[2 * i], win[2 * i + 1]);
    dist[i] = d;
    hit[i] = d <= add(a.r, b.r) ? 1 : 0;
  }
}

static int sort_pairs(ltsg_workspace* ws, const uint64_t* kin, uint64_t* kout, const int32_t* vin, int32_t* vout,
                      int64_t n, int end_bit, cudaStream_t st) {
  if (n <= 0) return LTSG_OK;
  size_t tmp = 0;
  LTSG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit, st));
  void* t = nullptr;
  LTSG_TRY(ws->get("bp_cub", tmp, &t));
  LTSG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, (int)n, 0, end_bit, st));
  return LTSG_OK;
}

static int sort_keys(ltsg_workspace* ws, const uint64_t* kin, uint64_t* kout, int64_t n, int end_bit,
                     cudaStream_t st) {
  if (n <= 0) return LTSG_OK;
  size_t tmp = 0;
  LTSG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, (int)n, 0, end_bit, st));
  void* t = nullptr;
  LTSG_TRY(ws->get("bp_cub", tmp, &t));
  LTSG_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, kin, kout, (int)n, 0, end_bit, st));
  return LTSG_OK;
}

static int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

template <typename T>
static int wsget(ltsg_workspace* ws, const char* name, int64_t count, T** out) {
  void* p = nullptr;
  LTSG_TRY(ws->get(name, (size_t)(count > 0 ? count : 1) * sizeof(T), &p));
  *out = (T*)p;
  return LTSG_OK;
}

}  // namespace bp
}  // namespace ltsg

using namespace ltsg;
using namespace ltsg::bp;

extern "C" {

int ltsg_broadphase(const ltsg_broad_input* in, ltsg_broad_output* out, ltsg_workspace* ws, void* stream) {
  if (!in || !out || !ws || in->n_particles < 0 || in->n_statics < 0 ||
      (in->n_particles > 0 && !in->particle) || (in->n_statics > 0 && !in->statics) || !(in->dt_max > 0.0) ||
      !(in->growth > 1.0)) {
    set_error("ltsg_broadphase: bad arguments");
    return LTSG_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n_p = in->n_particles, n_s = in->n_statics, n = n_p + n_s;
  out->n_edges = out->n_links = out->candidates = 0;
  out->launches = 0;
  if (n == 0) return LTSG_OK;
  if ((int64_t)n > (int64_t)1 << 30) {
    set_error("ltsg_broadphase: too many bodies (%d)", n);
    return LTSG_EINVAL;
  }
  cudaEvent_t e0 = ws->event(0), e1 = ws->event(1);
  LTSG_CUDA(cudaEventRecord(e0, st));
  Traj* traj;
  double *box, *sbox, *dts_tmp;
  uint64_t *key, *key_s;
  int32_t *idx, *idx_s, *sbody;
  unsigned long long* ctr;  // [0] candidates, [1] edges, [2] links
  LTSG_TRY(wsget(ws, "bp_traj", n, &traj));
  LTSG_TRY(wsget(ws, "bp_box", 6 * (int64_t)n, &box));
  LTSG_TRY(wsget(ws, "bp_sbox", 6 * (int64_t)n, &sbox));
  LTSG_TRY(wsget(ws, "bp_key", n, &key));
  LTSG_TRY(wsget(ws, "bp_key_s", n, &key_s));
  LTSG_TRY(wsget(ws, "bp_idx", n, &idx));
  LTSG_TRY(wsget(ws, "bp_idx_s", n, &idx_s));
  LTSG_TRY(wsget(ws, "bp_sbody", n, &sbody));
  LTSG_TRY(wsget(ws, "bp_ctr", 4, &ctr));
  double* dts = out->dts;
  if (!dts) {
    LTSG_TRY(wsget(ws, "bp_dts", n_p, &dts_tmp));
    dts = dts_tmp;
  }
  LTSG_CUDA(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), st));
  k_bp_traj<<<grid_for(n, 128), 128, 0, st>>>(in->particle, in->statics, n_p, n_s, in->dt_max, in->growth, traj,
                                              box, dts, key, idx);
  LTSG_CHECK_LAUNCH();
  ++out->launches;
  LTSG_TRY(sort_pairs(ws, key, key_s, idx, idx_s, n, 64, st));
  ++out->launches;
  k_bp_gather<<<grid_for(n, 128), 128, 0, st>>>(box, idx_s, n, sbox, sbody);
  LTSG_CHECK_LAUNCH();
  ++out->launches;

  // Check 1: candidates into a list sized from the last call; re-run once
  // with the exact size on overflow
  const int n_tiles = (n + kTile - 1) / kTile;
  const int tpc = 8;
  dim3 grid(n_tiles, (n_tiles + tpc - 1) / tpc);
  unsigned long long h_ctr[4] = {0, 0, 0, 0};
  int64_t cap = std::max<int64_t>((int64_t)ws->hint_bp_cand, 16 * (int64_t)n);
  Cand* cand = nullptr;
  for (int attempt = 0;; ++attempt) {
    LTSG_TRY(wsget(ws, "bp_cand", cap, &cand));
    LTSG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    k_bp_sweep<<<grid, kTile, 0, st>>>(sbox, sbody, n, n_p, tpc, cand, ctr, (unsigned long long)cap);
    LTSG_CHECK_LAUNCH();
    ++out->launches;
    LTSG_CUDA(cudaMemcpyAsync(h_ctr, ctr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    LTSG_CUDA(cudaStreamSynchronize(st));
    if ((int64_t)h_ctr[0] <= cap) break;
    cap = (int64_t)h_ctr[0] + (int64_t)h_ctr[0] / 4 + 64;
    if (attempt > 0) {
      set_error("ltsg_broadphase: candidate list overflow");
      return LTSG_ECAPACITY;
    }
  }
  const int64_t n_cand = (int64_t)h_ctr[0];
  ws->hint_bp_cand = std::max(ws->hint_bp_cand, (size_t)(n_cand + n_cand / 4));
  out->candidates = n_cand;

  // Check 2 and emission
  uint64_t *ekey, *ekey_s, *lkey, *lkey_s;
  double* ewin;
  int32_t *eperm, *eperm_s;
  LTSG_TRY(wsget(ws, "bp_ekey", n_cand, &ekey));
  LTSG_TRY(wsget(ws, "bp_ekey_s", n_cand, &ekey_s));
  LTSG_TRY(wsget(ws, "bp_lkey", n_cand, &lkey));
  LTSG_TRY(wsget(ws, "bp_lkey_s", n_cand, &lkey_s));
  LTSG_TRY(wsget(ws, "bp_ewin", 2 * n_cand, &ewin));
  LTSG_TRY(wsget(ws, "bp_eperm", n_cand, &eperm));
  LTSG_TRY(wsget(ws, "bp_eperm_s", n_cand, &eperm_s));
  if (n_cand > 0) {
    const int blocks = std::min(grid_for(n_cand, 128), 148 * 16);
    k_bp_tube<<<blocks, 128, 0, st>>>(cand, ctr, traj, in->particle, dts, n_p, n_s, ekey, ewin, eperm, ctr + 1, lkey,
                                      ctr + 2);
    LTSG_CHECK_LAUNCH();
    ++out->launches;
  }
  LTSG_CUDA(cudaMemcpyAsync(h_ctr + 1, ctr + 1, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  const int64_t n_e = (int64_t)h_ctr[1], n_l = (int64_t)h_ctr[2];
  out->n_edges = n_e;
  out->n_links = n_l;
  if (n_e > out->cap_edges || n_l > out->cap_links) {
    set_error("ltsg_broadphase: %lld edges / %lld links exceed the output capacity (%lld / %lld)",
              (long long)n_e, (long long)n_l, (long long)out->cap_edges, (long long)out->cap_links);
    return LTSG_ECAPACITY;
  }
  // edges in the reference's dict order (its sorted(candidates) walk: sorted
  // (index_a, index_b)); static links per particle in ascending static id
  if (n_e > 0)
    LTSG_TRY(sort_pairs(ws, ekey, ekey_s, eperm, eperm_s, n_e, bits_for((uint64_t)n_p * (uint64_t)n_p), st));
  if (n_l > 0)
    LTSG_TRY(sort_keys(ws, lkey, lkey_s, n_l, bits_for((uint64_t)n_p * (uint64_t)n_s), st));
  if (n_e > 0 || n_l > 0) {
    out->launches += (n_e > 0) + (n_l > 0);
    const int64_t m = std::max(n_e, n_l);
    k_bp_emit<<<grid_for(m, 128), 128, 0, st>>>(ekey_s, eperm_s, ewin, n_e, n_p, out->edge, out->window, lkey_s,
                                                n_l, n_s, out->link);
    LTSG_CHECK_LAUNCH();
    ++out->launches;
  }
  LTSG_CUDA(cudaEventRecord(e1, st));
  LTSG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  LTSG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  out->ms = (double)ms;
  return LTSG_OK;
}

int ltsg_tube_rows(const double* t1, const double* c1, const double* r1, const int32_t* nt1, const double* t2,
                   const double* c2, const double* r2, const int32_t* nt2, const double* win, int64_t n,
                   double* dist, int32_t* hit, void* stream) {
  if (n < 0 || (n > 0 && (!t1 || !c1 || !r1 || !nt1 || !t2 || !c2 || !r2 || !nt2 || !win || !dist || !hit))) {
    set_error("ltsg_tube_rows: bad arguments");
    return LTSG_EINVAL;
  }
  if (n == 0) return LTSG_OK;
  k_bp_tube_rows<<<std::min(grid_for(n, 128), 148 * 16), 128, 0, (cudaStream_t)stream>>>(
      t1, c1, r1, nt1, t2, c2, r2, nt2, win, n, dist, hit);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

}  // extern "C"
