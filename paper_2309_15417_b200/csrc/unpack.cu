// Compact tree upload: rebuild the 16-slot triangle records of ltsg_scene
// from the host's compact image (include/ltsgpu.h, ltsg_tree_upload).
//
// Slots 0..11 are bit-identical to packing.pack_tree's host build:
//   0..8  corners (copied: fine-level corners are mesh-vertex rows)
//   9     epsilon (copied)
//   10    arm = max over corners of norm(corner), numpy's row order
//         sqrt((x*x + y*y) + z*z) (ccd._Motion.arm, ccd.py:108-114)
//   11    (int32 first child, int32 count), 0 on the fine level
// Slots 12..15 are cull data (sphere centre, inflated radius, -1 for
// slivers); they only have to be conservative, not bit-identical.
#include "common.cuh"
#include "geom.cuh"

namespace ltsg {

constexpr int kUnpackThreads = 128;
constexpr int kRec = 16;
constexpr double kSliverCond = 1e4;  // packing.CULL_COND

__global__ void __launch_bounds__(kUnpackThreads)
k_unpack_trees(ltsg_tree_upload up, double* __restrict__ tris) {
  __shared__ double s_out[kUnpackThreads * kRec];
  for (int t = blockIdx.x; t < up.n_trees; t += gridDim.x) {
    const int64_t* row = up.table + 8 * (int64_t)t;
    const int64_t rec_off = row[0], n_fine = row[1], n_coarse = row[2], vert_off = row[3], vidx_off = row[4],
                  coarse_off = row[5], eps_off = row[6], eps_mode = row[7];
    const int64_t n = n_fine + n_coarse;
    for (int64_t j0 = 0; j0 < n; j0 += kUnpackThreads) {
      const int m = (int)min((int64_t)kUnpackThreads, n - j0);
      if (threadIdx.x < m) {
        const int64_t j = j0 + threadIdx.x;
        double c[9];
        double eps;
        int2 kid = make_int2(0, 0);
        if (j < n_fine) {
          const int32_t* vi = up.vidx + 3 * (vidx_off + j);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double* v = up.verts + 3 * (vert_off + vi[k]);
            c[3 * k] = v[0];
            c[3 * k + 1] = v[1];
            c[3 * k + 2] = v[2];
          }
          eps = up.eps[eps_off + (eps_mode ? j : 0)];
        } else {
          const int64_t q = coarse_off + (j - n_fine);
          const double* src = up.coarse + 9 * q;
#pragma unroll
          for (int k = 0; k < 9; ++k) c[k] = src[k];
          eps = up.eps[eps_off + (eps_mode ? j : 1 + (j - n_fine))];
          kid = reinterpret_cast<const int2*>(up.kids)[q];
        }
        double* r = s_out + threadIdx.x * kRec;
#pragma unroll
        for (int k = 0; k < 9; ++k) r[k] = c[k];
        r[9] = eps;
        double arm = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double nk = __dsqrt_rn(add(add(mul(c[3 * k], c[3 * k]), mul(c[3 * k + 1], c[3 * k + 1])),
                                           mul(c[3 * k + 2], c[3 * k + 2])));
          arm = k ? fmax(arm, nk) : nk;  // np.max over the 3 norms
        }
        r[10] = arm;
        *reinterpret_cast<int2*>(r + 11) = kid;
        // cull sphere: centroid, radius inflated by 1e-12, -1 for slivers
        const double cx = (c[0] + c[3] + c[6]) / 3.0, cy = (c[1] + c[4] + c[7]) / 3.0,
                     cz = (c[2] + c[5] + c[8]) / 3.0;
        double r2 = 0.0, l2 = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double dx = c[3 * k] - cx, dy = c[3 * k + 1] - cy, dz = c[3 * k + 2] - cz;
          r2 = fmax(r2, fma(dx, dx, fma(dy, dy, dz * dz)));
          const int k1 = (k + 1) % 3;
          const double ex = c[3 * k1] - c[3 * k], ey = c[3 * k1 + 1] - c[3 * k + 1], ez = c[3 * k1 + 2] - c[3 * k + 2];
          l2 = fmax(l2, fma(ex, ex, fma(ey, ey, ez * ez)));
        }
        const double e0x = c[3] - c[0], e0y = c[4] - c[1], e0z = c[5] - c[2];
        const double e2x = c[6] - c[0], e2y = c[7] - c[1], e2z = c[8] - c[2];
        const double nx = fma(e0y, e2z, -e0z * e2y), ny = fma(e0z, e2x, -e0x * e2z), nz = fma(e0x, e2y, -e0y * e2x);
        const double area2 = sqrt(fma(nx, nx, fma(ny, ny, nz * nz)));
        const bool ok = area2 > 0.0 && l2 <= kSliverCond * area2;
        r[12] = cx;
        r[13] = cy;
        r[14] = cz;
        r[15] = ok ? sqrt(r2) * (1.0 + 1e-12) : -1.0;
      }
      __syncthreads();
      double2* dst = reinterpret_cast<double2*>(tris + (size_t)(rec_off + j0) * kRec);
      const double2* src = reinterpret_cast<const double2*>(s_out);
      for (int k = threadIdx.x; k < m * kRec / 2; k += kUnpackThreads) dst[k] = src[k];
      __syncthreads();
    }
  }
}

}  // namespace ltsg

extern "C" int ltsg_unpack_trees(const ltsg_tree_upload* up, double* tris_out, void* stream) {
  using namespace ltsg;
  if (!up || !tris_out || up->n_trees < 0 || (up->n_trees > 0 && (!up->table || !up->eps))) {
    set_error("ltsg_unpack_trees: invalid arguments");
    return LTSG_EINVAL;
  }
  if (up->n_trees == 0) return LTSG_OK;
  const int grid = (int)std::min<int64_t>(up->n_trees, 148 * 16);
  k_unpack_trees<<<grid, kUnpackThreads, 0, (cudaStream_t)stream>>>(*up, tris_out);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}
