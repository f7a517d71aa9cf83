// Row-batched geometry kernels (drop-ins for ltsdem.kernels / ccd row
// helpers), error state and the workspace.
#include "common.cuh"
#include "geom.cuh"
#include "dist_staged.cuh"
#include "dist_tile.cuh"

#include <atomic>
#include <cstdint>
#include <cstring>

namespace ltsg {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

__device__ __forceinline__ V3 ld3(const double* p, int64_t i) {
  return V3{p[3 * i], p[3 * i + 1], p[3 * i + 2]};
}
__device__ __forceinline__ void st3(double* p, int64_t i, V3 v) {
  p[3 * i] = v.x;
  p[3 * i + 1] = v.y;
  p[3 * i + 2] = v.z;
}
__device__ __forceinline__ Tri ldtri(const double* p, int64_t i) {
  Tri t;
  const double* q = p + 9 * i;
#pragma unroll
  for (int k = 0; k < 3; ++k) t.v[k] = V3{q[3 * k], q[3 * k + 1], q[3 * k + 2]};
  return t;
}

__global__ void k_point_triangle(const double* p, const double* a, const double* b, const double* c,
                                 int64_t n, double* dist, double* closest) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const V3 P = ld3(p, i), A = ld3(a, i), B = ld3(b, i), C = ld3(c, i);
    V3 q;
    int reg;
    const double sq = point_triangle_sq<false, true>(P, A, B, C, B - A, C - A, C - B, &q, &reg);
    dist[i] = __dsqrt_rn(sq);
    if (closest) st3(closest, i, q);
  }
}

__global__ void k_segment_segment(const double* p1, const double* q1, const double* p2,
                                  const double* q2, int64_t n, double* dist, double* c1,
                                  double* c2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const V3 P1 = ld3(p1, i), P2 = ld3(p2, i);
    const V3 u = ld3(q1, i) - P1, w = ld3(q2, i) - P2;
    V3 x1, x2;
    const double sq = segment_segment_sq<true>(P1, u, dot_simd(u, u), P2, w, dot_simd(w, w), &x1, &x2);
    dist[i] = __dsqrt_rn(sq);
    if (c1) st3(c1, i, x1);
    if (c2) st3(c2, i, x2);
  }
}

// ccd._feature_distances per row with the distance of dist_tile.cuh: both
// triangles' per-triangle constants (edges, |e|^2, reciprocals) staged per
// lane in shared memory.  The loop is warp-uniform (lanes past the end
// evaluate a duplicate row) because the distance votes across the warp.
#ifndef LTSG_ROWS_STAGED
#define LTSG_ROWS_STAGED 0
#endif
__global__ void __launch_bounds__(128, 4) k_feature_distances(const double* ta, const double* tb, int64_t n,
                                                           double* dist) {
#if LTSG_ROWS_STAGED
  __shared__ double s_stage[kStaged * 128];
  const Staged<128> st{s_stage + threadIdx.x};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    stage_pair(st, ldtri(ta, i), ldtri(tb, i));
    dist[i] = __dsqrt_rn(staged_dist_sq(st));
  }
#else
  __shared__ double s_stage[2 * kTileASlots * 128];
  double* sa = s_stage + threadIdx.x;
  double* sb = s_stage + kTileASlots * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); w0 < n; w0 += stride) {
    const int64_t i = w0 + lane;  // w0 is the same on every lane: the loop is warp-uniform
    const int64_t r = i < n ? i : n - 1;
    const TriReg A = tri_reg(ldtri(ta, r), 0.0), B = tri_reg(ldtri(tb, r), 0.0);
    tri_store_soa<128>(sa, A);
    tri_store_soa<128>(sb, B);
    const double d = __dsqrt_rn(exact_dist_sq(SmemTri<128>{sa}, SmemTri<128>{sb}, A.regular && B.regular));
    if (i < n) dist[i] = d;
  }
#endif
}

__global__ void k_closest_feature(const double* ta, const double* tb, int64_t n, double* dist,
                                  double* pa, double* pb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    V3 a, b;
    dist[i] = closest_feature(ldtri(ta, i), ldtri(tb, i), &a, &b);
    st3(pa, i, a);
    st3(pb, i, b);
  }
}

__global__ void k_overlap_centroid(const double* ta, const double* tb, const double* nrm, int64_t n,
                                   double* out, int32_t* has) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    V3 c{0.0, 0.0, 0.0};
    const bool ok = overlap_centroid(ldtri(ta, i), ldtri(tb, i), ld3(nrm, i), &c);
    st3(out, i, c);
    has[i] = ok ? 1 : 0;
  }
}

// Independent DFMA chains (8 per thread) keep every FP64 pipe busy.
__global__ void __launch_bounds__(256) k_fp64_peak(double* sink, int iters, double seed) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed + threadIdx.x * 1e-9 + k;
  const double a = 0.999999999, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) sink[0] = s;  // keep the chains alive
}

static int row_grid(int64_t n) {
  int64_t g = (n + 127) / 128;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return (int)g;
}

}  // namespace ltsg

using namespace ltsg;

extern "C" {

const char* ltsg_last_error(void) { return g_err; }
int ltsg_version(void) { return 1; }

int ltsg_point_triangle_closest(const double* p, const double* a, const double* b, const double* c,
                                int64_t n, double* dist, double* closest, void* stream) {
  if (n < 0 || (n > 0 && (!p || !a || !b || !c || !dist))) {
    set_error("ltsg_point_triangle_closest: bad arguments");
    return LTSG_EINVAL;
  }
  if (n == 0) return LTSG_OK;
  k_point_triangle<<<row_grid(n), 128, 0, (cudaStream_t)stream>>>(p, a, b, c, n, dist, closest);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

int ltsg_segment_segment_closest(const double* p1, const double* q1, const double* p2,
                                 const double* q2, int64_t n, double* dist, double* c1, double* c2,
                                 void* stream) {
  if (n < 0 || (n > 0 && (!p1 || !q1 || !p2 || !q2 || !dist))) {
    set_error("ltsg_segment_segment_closest: bad arguments");
    return LTSG_EINVAL;
  }
  if (n == 0) return LTSG_OK;
  k_segment_segment<<<row_grid(n), 128, 0, (cudaStream_t)stream>>>(p1, q1, p2, q2, n, dist, c1, c2);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

int ltsg_feature_distances(const double* ta, const double* tb, int64_t n, double* dist,
                           void* stream) {
  if (n < 0 || (n > 0 && (!ta || !tb || !dist))) {
    set_error("ltsg_feature_distances: bad arguments");
    return LTSG_EINVAL;
  }
  if (n == 0) return LTSG_OK;
  k_feature_distances<<<row_grid(n), 128, 0, (cudaStream_t)stream>>>(ta, tb, n, dist);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

int ltsg_closest_feature(const double* ta, const double* tb, int64_t n, double* dist, double* pa,
                         double* pb, void* stream) {
  if (n < 0 || (n > 0 && (!ta || !tb || !dist || !pa || !pb))) {
    set_error("ltsg_closest_feature: bad arguments");
    return LTSG_EINVAL;
  }
  if (n == 0) return LTSG_OK;
  k_closest_feature<<<row_grid(n), 128, 0, (cudaStream_t)stream>>>(ta, tb, n, dist, pa, pb);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

int ltsg_overlap_centroid(const double* ta, const double* tb, const double* normal, int64_t n,
                          double* centroid, int32_t* has, void* stream) {
  if (n < 0 || (n > 0 && (!ta || !tb || !normal || !centroid || !has))) {
    set_error("ltsg_overlap_centroid: bad arguments");
    return LTSG_EINVAL;
  }
  if (n == 0) return LTSG_OK;
  k_overlap_centroid<<<row_grid(n), 128, 0, (cudaStream_t)stream>>>(ta, tb, normal, n, centroid, has);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

int ltsg_fp64_peak(double* tflops, double* ms, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* sink = nullptr;
  LTSG_CUDA(cudaMalloc(&sink, sizeof(double)));
  int dev = 0, sms = 0;
  LTSG_CUDA(cudaGetDevice(&dev));
  LTSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  k_fp64_peak<<<blocks, threads, 0, st>>>(sink, 256, 1.0);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  k_fp64_peak<<<blocks, threads, 0, st>>>(sink, iters, 1.0);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float m = 0.f;
  cudaEventElapsedTime(&m, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  LTSG_CUDA(cudaGetLastError());
  const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  *ms = m;
  *tflops = flops / (m * 1e-3) / 1e12;
  return LTSG_OK;
}

ltsg_workspace* ltsg_workspace_create(int64_t budget_bytes) {
  ltsg_workspace* ws = new ltsg_workspace();
  cudaGetDevice(&ws->device);
  // 0 = no per-workspace cap: only the process-wide pool (below) applies
  ws->budget = budget_bytes > 0 ? (size_t)budget_bytes : SIZE_MAX;
  return ws;
}

void ltsg_workspace_destroy(ltsg_workspace* ws) { delete ws; }

int64_t ltsg_workspace_bytes(const ltsg_workspace* ws) { return ws ? (int64_t)ws->total : 0; }

}  // extern "C"

// Process-wide budget shared by every workspace (one per engine thread): 75%
// of the device memory free when the first workspace allocates.  N threads
// therefore cannot jointly claim more than the device has; a request beyond
// it is a capacity condition (LTSG_ECAPACITY: the host splits the batch),
// while a failing cudaMalloc inside the budget is a genuine out-of-memory
// (LTSG_ENOMEM: not retried by splitting).
static std::atomic<size_t> g_pool_used{0};
static std::atomic<size_t> g_pool_budget{0};

static size_t pool_budget() {
  size_t b = g_pool_budget.load();
  if (b == 0) {
    size_t free_b = 0, total_b = 0;
    b = cudaMemGetInfo(&free_b, &total_b) == cudaSuccess ? (size_t)(0.75 * (double)free_b) : ((size_t)8 << 30);
    size_t zero = 0;
    if (!g_pool_budget.compare_exchange_strong(zero, b)) b = zero;
  }
  return b;
}

static bool pool_reserve(size_t bytes) {
  const size_t budget = pool_budget();
  size_t cur = g_pool_used.load();
  while (true) {
    if (cur + bytes > budget) return false;
    if (g_pool_used.compare_exchange_weak(cur, cur + bytes)) return true;
  }
}

static void pool_release(size_t bytes) { g_pool_used.fetch_sub(bytes); }

int ltsg_workspace::get(const char* name, size_t bytes, void** out, bool keep) {
  Buf& b = bufs[name];
  if (bytes == 0) bytes = 256;
  if (b.bytes >= bytes) {
    *out = b.ptr;
    return LTSG_OK;
  }
  size_t want = bytes + bytes / 2;
  if (total - b.bytes + want > budget) want = bytes;
  if (total - b.bytes + want > budget) {
    set_error("workspace budget exceeded: slot %s needs %zu bytes (total %zu, budget %zu)", name,
              bytes, total, budget);
    return LTSG_ECAPACITY;
  }
  // the old buffer stays allocated while a kept one is copied: reserve both
  if (!pool_reserve(want)) {
    want = bytes;
    if (!pool_reserve(want)) {
      set_error("device memory pool exhausted: slot %s needs %zu bytes (pool %zu of %zu in use)", name, bytes,
                g_pool_used.load(), pool_budget());
      return LTSG_ECAPACITY;
    }
  }
  void* p = nullptr;
  cudaError_t err = cudaMalloc(&p, want);
  if (err != cudaSuccess) {
    cudaGetLastError();
    pool_release(want);
    set_error("cudaMalloc(%zu) for %s failed: %s", want, name, cudaGetErrorString(err));
    return LTSG_ENOMEM;
  }
  if (b.ptr) {
    if (keep) cudaMemcpy(p, b.ptr, b.bytes, cudaMemcpyDeviceToDevice);
    cudaFree(b.ptr);
    pool_release(b.bytes);
  }
  total = total - b.bytes + want;
  b.ptr = p;
  b.bytes = want;
  *out = p;
  return LTSG_OK;
}

ltsg_workspace::~ltsg_workspace() {
  for (auto& kv : bufs)
    if (kv.second.ptr) {
      cudaFree(kv.second.ptr);
      pool_release(kv.second.bytes);
    }
  for (auto e : events)
    if (e) cudaEventDestroy(e);
}
