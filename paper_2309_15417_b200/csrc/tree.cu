// Surrogate-tree construction on sm_100a: ltsdem.surrogate.build_surrogate_tree
// (surrogate.py:71-119) for many meshes per call, bit-identical to the
// reference on the build host (the narrow phase's on-device
// input format).
//
// One coarse level of every mesh per round (levels depend on the previous
// one), three steps per round:
//   k_tree_codes  one block per mesh: triangle centroids (the sequential
//                 `corners.mean(axis=1)`), their bounding box, 10-bit
//                 quantisation and the 30-bit Morton code of
//                 kernels.morton_order (kernels.py:118-135).  Key =
//                 (mesh rank in the round << 30) | code.
//   cub radix sort of (key, triangle) pairs over the round: radix sort is
//                 stable, so equal codes keep ascending triangle order --
//                 numpy's argsort(kind="stable").
//   k_tree_fit    one thread per group of `fanout` consecutive triangles in
//                 Morton order: _fit_parent_triangle (surrogate.py:49-68) --
//                 centroid, the LAPACK plane basis (lapack3.cuh), projections
//                 in OpenBLAS dgemv order, padded bounds, the parent triangle
//                 -- then the halo cover max(dist + child eps) + 1e-12 with
//                 kernels.point_triangle_closest (surrogate.py:100-113) and the
//                 sorted child list (surrogate.py:115).
//
// Rounding: -fmad=false plus explicit __d*_rn / __fma_rn where the reference
// (numpy elementwise vs OpenBLAS) fuses.  Groups are independent, so the
// thread-per-group fit needs no cross-lane order.
#include "common.cuh"
#include "geom.cuh"
#include "lapack3.cuh"

#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>

namespace ltsg {
namespace tree {

constexpr int kStepCols = 6;  // [in_off, n_in, out_off, n_out, key_off, group_off]
constexpr int kMaxFanout = lapack::kLda / 3;

__device__ __forceinline__ void tri_centroid(const double* r, double c[3]) {
  // corners.mean(axis=1): ((c0 + c1) + c2) / 3
  for (int a = 0; a < 3; ++a) c[a] = dv(add(add(r[a], r[3 + a]), r[6 + a]), 3.0);
}

__global__ void __launch_bounds__(256) k_tree_codes(const double* __restrict__ rec, const int64_t* __restrict__ steps,
                                                    int s0, uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  __shared__ double red[2][3][256 / 32];
  const int64_t* st = steps + (int64_t)(s0 + blockIdx.x) * kStepCols;
  const int64_t in_off = st[0], n_in = st[1], key_off = st[4];
  double lo[3] = {CUDART_INF, CUDART_INF, CUDART_INF}, hi[3] = {-CUDART_INF, -CUDART_INF, -CUDART_INF};
  for (int64_t t = threadIdx.x; t < n_in; t += blockDim.x) {
    double c[3];
    tri_centroid(rec + 9 * (in_off + t), c);
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], c[a]);
      hi[a] = fmax(hi[a], c[a]);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if (lane == 0) {
      red[0][a][warp] = lo[a];
      red[1][a][warp] = hi[a];
    }
  }
  __syncthreads();
  double scale[3];
  for (int a = 0; a < 3; ++a) {
    double l = red[0][a][0], h = red[1][a][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      l = fmin(l, red[0][a][w]);
      h = fmax(h, red[1][a][w]);
    }
    lo[a] = l;
    double span = sub(h, l);
    if (span <= 0.0) span = 1.0;
    scale[a] = dv(1023.0, span);  // (2**bits - 1) / span
  }
  const uint64_t hib = (uint64_t)blockIdx.x << 30;
  for (int64_t t = threadIdx.x; t < n_in; t += blockDim.x) {
    double c[3];
    tri_centroid(rec + 9 * (in_off + t), c);
    uint64_t q[3];
    for (int a = 0; a < 3; ++a) q[a] = (uint64_t)mul(sub(c[a], lo[a]), scale[a]);  // astype(np.uint64)
    uint64_t code = 0;
    for (int i = 0; i < 10; ++i)
      for (int a = 0; a < 3; ++a) code |= ((q[a] >> i) & 1ull) << (3 * i + a);
    key[key_off + t] = hib | code;
    val[key_off + t] = (int32_t)t;
  }
}

__device__ __forceinline__ int find_step(const int64_t* steps, int s0, int s1, int64_t gid) {
  // last step of [s0, s1) with group_off <= gid
  int lo = s0, hi = s1 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (steps[(int64_t)mid * kStepCols + 5] <= gid)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(128) k_tree_fit(double* __restrict__ rec, double* __restrict__ eps,
                                                  int32_t* __restrict__ kids, const int64_t* __restrict__ steps,
                                                  int s0, int s1, int64_t n_groups, const int32_t* __restrict__ order,
                                                  int fanout, int32_t* __restrict__ status) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n_groups) return;
  const int s = find_step(steps, s0, s1, gid);
  const int64_t* st = steps + (int64_t)s * kStepCols;
  const int64_t in_off = st[0], n_in = st[1], out_off = st[2], key_off = st[4];
  const int64_t g = gid - st[5];
  const int64_t k0 = g * fanout;
  const int k = (int)min((int64_t)fanout, n_in - k0);
  int idx[kMaxFanout];
  for (int j = 0; j < k; ++j) idx[j] = order[key_off + k0 + j];
  const int m = 3 * k;
  // points (m, 3): the group's triangles in Morton order, corners 0, 1, 2
  double P[3 * kMaxFanout][3];
  for (int j = 0; j < k; ++j) {
    const double* r = rec + 9 * (in_off + idx[j]);
    for (int c = 0; c < 3; ++c)
      for (int a = 0; a < 3; ++a) P[3 * j + c][a] = r[3 * c + a];
  }
  // points.mean(axis=0): sequential row sum, then / m
  double cen[3];
  for (int a = 0; a < 3; ++a) {
    double acc = P[0][a];
    for (int i = 1; i < m; ++i) acc = add(acc, P[i][a]);
    cen[a] = dv(acc, (double)m);
  }
  double A[3 * lapack::kLda];  // rel, column-major (overwritten by the SVD)
  double spread = 0.0;
  for (int i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) {
      P[i][a] = sub(P[i][a], cen[a]);  // rel
      A[i + lapack::kLda * a] = P[i][a];
      spread = fmax(spread, fabs(P[i][a]));
    }
  double VT[9];
  if (!lapack::svd_vt(A, m, VT)) {
    atomicExch(status, 1);
    return;
  }
  const V3 u{VT[0], VT[3], VT[6]}, v{VT[1], VT[4], VT[7]};
  // su = rel @ u (OpenBLAS dgemv_t tail of three rows), likewise sv
  double lo_u = CUDART_INF, hi_u = -CUDART_INF, lo_v = CUDART_INF, hi_v = -CUDART_INF;
  for (int i = 0; i < m; ++i) {
    const double su = add(0.0, fma_(P[i][2], u.z, fma_(P[i][0], u.x, mul(P[i][1], u.y))));
    const double sv = add(0.0, fma_(P[i][2], v.z, fma_(P[i][0], v.x, mul(P[i][1], v.y))));
    lo_u = fmin(lo_u, su);
    hi_u = fmax(hi_u, su);
    lo_v = fmin(lo_v, sv);
    hi_v = fmax(hi_v, sv);
  }
  if (spread == 0.0) spread = 1.0;
  const double pad = fmax(1e-9, mul(1e-6, spread));
  lo_u = sub(lo_u, pad);
  hi_u = add(hi_u, pad);
  lo_v = sub(lo_v, pad);
  hi_v = add(hi_v, pad);
  const double w = sub(hi_u, lo_u), h = sub(hi_v, lo_v);
  const V3 c0{cen[0], cen[1], cen[2]};
  const V3 p0 = (c0 + scale(u, lo_u)) + scale(v, lo_v);
  const V3 p1 = p0 + scale(u, mul(2.0, w));
  const V3 p2 = p0 + scale(v, mul(2.0, h));
  // halo cover: max over the group's corners of dist(corner, parent) + child eps
  const V3 ab = p1 - p0, ac = p2 - p0, bc = p2 - p1;
  double cover = -CUDART_INF;
  for (int j = 0; j < k; ++j) {
    const double ce = eps[in_off + idx[j]];
    for (int c = 0; c < 3; ++c) {
      const double* r = rec + 9 * (in_off + idx[j]) + 3 * c;
      const V3 pt{r[0], r[1], r[2]};
      const double d = __dsqrt_rn(point_triangle_sq<false, false>(pt, p0, p1, p2, ab, ac, bc));
      cover = fmax(cover, add(d, ce));
    }
  }
  double* out = rec + 9 * (out_off + g);
  out[0] = p0.x;
  out[1] = p0.y;
  out[2] = p0.z;
  out[3] = p1.x;
  out[4] = p1.y;
  out[5] = p1.z;
  out[6] = p2.x;
  out[7] = p2.y;
  out[8] = p2.z;
  eps[out_off + g] = add(cover, 1e-12);
  // np.sort(group)
  for (int a = 1; a < k; ++a)
    for (int b = a; b > 0 && idx[b - 1] > idx[b]; --b) {
      const int t = idx[b];
      idx[b] = idx[b - 1];
      idx[b - 1] = t;
    }
  for (int j = 0; j < k; ++j) kids[in_off + k0 + j] = idx[j];
}

template <class T>
static int wsget(ltsg_workspace* ws, const char* name, int64_t count, T** out) {
  void* p = nullptr;
  LTSG_TRY(ws->get(name, (size_t)(count > 0 ? count : 1) * sizeof(T), &p));
  *out = (T*)p;
  return LTSG_OK;
}

}  // namespace tree
}  // namespace ltsg

using namespace ltsg;
using namespace ltsg::tree;

extern "C" {

int ltsg_build_trees(ltsg_tree_build* b, ltsg_workspace* ws, void* stream) {
  if (!b || !ws || !b->rec || !b->eps || !b->kids || !b->steps || !b->level_steps || !b->level_keys ||
      !b->level_groups || b->n_levels < 0 || b->fanout < 2 || b->fanout > kMaxFanout) {
    set_error("ltsg_build_trees: bad arguments (fanout must be 2..%d)", kMaxFanout);
    return LTSG_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int64_t max_keys = 0;
  for (int l = 0; l < b->n_levels; ++l) max_keys = std::max(max_keys, b->level_keys[l]);
  uint64_t *key, *key_s;
  int32_t *val, *val_s, *status;
  LTSG_TRY(wsget(ws, "tree_key", max_keys, &key));
  LTSG_TRY(wsget(ws, "tree_key_s", max_keys, &key_s));
  LTSG_TRY(wsget(ws, "tree_val", max_keys, &val));
  LTSG_TRY(wsget(ws, "tree_val_s", max_keys, &val_s));
  LTSG_TRY(wsget(ws, "tree_status", 1, &status));
  LTSG_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  int launches = 1;
  for (int l = 0; l < b->n_levels; ++l) {
    const int s0 = (int)b->level_steps[l], s1 = (int)b->level_steps[l + 1];
    const int ns = s1 - s0;
    const int64_t nk = b->level_keys[l], ng = b->level_groups[l];
    if (ns <= 0 || nk <= 0) continue;
    if (ns > (1 << 26) || nk > INT32_MAX) {
      set_error("ltsg_build_trees: level %d too large (%d meshes, %lld triangles)", l + 1, ns, (long long)nk);
      return LTSG_EINVAL;
    }
    k_tree_codes<<<ns, 256, 0, st>>>(b->rec, b->steps, s0, key, val);
    LTSG_CHECK_LAUNCH();
    int end_bit = 30;
    while ((1 << (end_bit - 30)) < ns) ++end_bit;
    size_t tmp = 0;
    cub::DoubleBuffer<uint64_t> kb(key, key_s);
    cub::DoubleBuffer<int32_t> vb(val, val_s);
    LTSG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int)nk, 0, end_bit, st));
    void* t = nullptr;
    LTSG_TRY(ws->get("tree_cub", tmp, &t));
    LTSG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, (int)nk, 0, end_bit, st));
    k_tree_fit<<<grid_for(ng, 128), 128, 0, st>>>(b->rec, b->eps, b->kids, b->steps, s0, s1, ng, vb.Current(),
                                                 b->fanout, status);
    LTSG_CHECK_LAUNCH();
    launches += 3;
  }
  b->launches = launches;
  int32_t h_status = 0;
  LTSG_CUDA(cudaMemcpyAsync(&h_status, status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  LTSG_CUDA(cudaStreamSynchronize(st));
  if (h_status) {
    set_error("ltsg_build_trees: the plane-fit SVD did not converge for some group");
    return LTSG_EINVAL;
  }
  return LTSG_OK;
}

}  // extern "C"
