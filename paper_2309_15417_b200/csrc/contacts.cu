// Contact consumers on sm_100a: the step after the narrow phase
// (ltsdem.contacts, contacts.py) for every cluster of a sweep in one launch.
//
//   k_solve      one warp per cluster: the contact arms (_contact_arm,
//                contacts.py:100-111: free flight to the contact time,
//                world inverse inertia rot Iinv rot^T, the arm from the
//                mass centre), the normal mobility and restitution bias
//                (:134-150), the greedy colour classes (color_contact_graph,
//                :58-78), then the relaxed sequential-impulse sweeps
//                (:157-190) class by class.  Contacts of one class touch
//                disjoint dynamic bodies (that is what the colouring
//                guarantees), so the lanes process a class's contacts at
//                once and the result is the reference's sequential one bit
//                for bit; `worst` is a max, which no order changes.
//   k_integrate  one warp per cluster: integrate_cluster (:225-253), each
//                member's free flight to its first contact, the post-impulse
//                velocities, free flight to the end of the step; then
//                apply_separation (:256-285) on lane 0 in the reference's
//                sorted body-pair order.
//
// Rounding: elementwise numpy arithmetic is separately rounded (-fmad=false,
// explicit __d*_rn), `(3,3) @ (3,)` is OpenBLAS dgemv (dot_gemv),
// `(3,3) @ (3,3)` dgemm (an FMA chain over k), 1-D `@` / np.linalg.norm ddot
// (dot_blas).  The transcendental on the path is quaternions.advance's
// sin/cos for spinning bodies; without spin the results are bit-identical.
#include "common.cuh"
#include "geom.cuh"
#include "quat.cuh"

#include <math_constants.h>

#include <algorithm>

namespace ltsg {
namespace cs {

constexpr int kBody = 24;  // body record, see ltsgpu.h (ltsg_solve_input)
constexpr int kArm = 32;   // per contact scratch: see ArmRec

// per-contact arm scratch: [0..2] r_a [3..5] r_b [6..14] Iinv_a (world)
// [15..23] Iinv_b [24] inv_mass_a [25] inv_mass_b [26] k_normal [27] bias
__device__ __forceinline__ V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double* p, V3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}

__device__ __forceinline__ V3 gemv(const double* m, V3 v) {  // (3,3) @ (3,) through dgemv
  return V3{dot_gemv(V3{m[0], m[1], m[2]}, v), dot_gemv(V3{m[3], m[4], m[5]}, v), dot_gemv(V3{m[6], m[7], m[8]}, v)};
}

__device__ __forceinline__ void gemm(const double* a, const double* b, double* out) {  // dgemm, FMA chain over k
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      out[3 * i + j] = fma_(a[3 * i + 2], b[6 + j], fma_(a[3 * i + 1], b[3 + j], mul(a[3 * i], b[j])));
}

// _Arm.mobility (:92-97)
__device__ __forceinline__ double mobility(double inv_mass, V3 r, const double* inv_i, V3 d) {
  if (inv_mass == 0.0) return 0.0;
  const V3 rxd = cross(r, d);
  return add(inv_mass, dot_blas(d, cross(gemv(inv_i, rxd), r)));
}

// extrapolate_free_flight (state.py:89-99) of a body record's current
// snapshot: position and rotation after dt
__device__ __forceinline__ void flight(const double* rec, double dt, V3* pos, double q[4]) {
  *pos = ld3(rec) + scale(ld3(rec + 3), dt);
  advance(rec + 6, ld3(rec + 10), dt, q);
}

__device__ __forceinline__ int lowest_zero(unsigned long long m) { return __ffsll((long long)~m) - 1; }

struct SolveArgs {
  const double* body;
  const int64_t* off;
  const int32_t* side;
  const double* position;
  const double* normal;
  const double* t;
  double restitution, friction, relaxation, penalty, threshold;
  int32_t max_iterations;
  int32_t n_problems;
  // scratch
  double* arm;                 // n_contacts x kArm
  double* vel;                 // n_bodies x 6 (velocity, angular velocity)
  unsigned long long* cls;     // n_bodies: bitset of the colour classes (< 64) holding the body
  int32_t* order;              // n_contacts: contacts of a problem by class
  int32_t* class_off;          // n_contacts + n_problems: class segments per problem
  // outputs
  double* out_vel;
  double* out_ang;
  int32_t* touched;
  double* lam;
  double* fric;
  int32_t* color;
  int32_t* iterations;
  int32_t* converged;
};

__device__ __forceinline__ V3 rel_vel(const SolveArgs& A, int ia, int ib, V3 ra, V3 rb) {  // (:201-204)
  V3 va{0.0, 0.0, 0.0}, vb{0.0, 0.0, 0.0};
  if (ia >= 0) va = ld3(A.vel + 6 * (size_t)ia) + cross(ld3(A.vel + 6 * (size_t)ia + 3), ra);
  if (ib >= 0) vb = ld3(A.vel + 6 * (size_t)ib) + cross(ld3(A.vel + 6 * (size_t)ib + 3), rb);
  return va - vb;
}

__device__ __forceinline__ void apply_imp(const SolveArgs& A, int ia, int ib, const double* arm, V3 imp) {  // (:207-213)
  if (ia >= 0) {
    double* v = A.vel + 6 * (size_t)ia;
    st3(v, ld3(v) + scale(imp, arm[24]));
    st3(v + 3, ld3(v + 3) + gemv(arm + 6, cross(ld3(arm), imp)));
  }
  if (ib >= 0) {
    double* v = A.vel + 6 * (size_t)ib;
    st3(v, ld3(v) - scale(imp, arm[25]));
    st3(v + 3, ld3(v + 3) - gemv(arm + 15, cross(ld3(arm + 3), imp)));
  }
}

__device__ __forceinline__ double measure(int ia, int ib, const double* arm, V3 imp) {  // (:216-222)
  double m = norm_blas(imp);
  if (ia >= 0) m = fmax(m, norm_blas(cross(ld3(arm), imp)));
  if (ib >= 0) m = fmax(m, norm_blas(cross(ld3(arm + 3), imp)));
  return m;
}

__global__ void k_solve(SolveArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < A.n_problems; p += nw) {
    const int64_t c0 = A.off[p], c1 = A.off[p + 1];
    const int n = (int)(c1 - c0);
    if (n == 0) {
      if (lane == 0) {
        A.iterations[p] = 0;
        A.converged[p] = 1;
      }
      continue;
    }
    // ---- arms, mobility, bias (:134-150); every touched body starts at its
    // current velocity (identical writes from every contact that touches it)
    for (int k = lane; k < n; k += 32) {
      const int64_t c = c0 + k;
      const double tc = A.t[c];
      const V3 pc = ld3(A.position + 3 * c);
      const V3 nrm = ld3(A.normal + 3 * c);
      double* arm = A.arm + (size_t)c * kArm;
      for (int s = 0; s < 2; ++s) {
        const int b = A.side[2 * c + s];
        V3 r{0.0, 0.0, 0.0};
        double invm = 0.0, inv_i[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (b >= 0) {
          const double* rec = A.body + (size_t)b * kBody;
          const double dt = sub(tc, rec[13]);
          V3 pos;
          double q[4], rot[9], rt[9], tmp[9];
          flight(rec, dt, &pos, q);
          to_matrix(q, rot);
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) rt[3 * i + j] = rot[3 * j + i];
          gemm(rot, rec + 15, tmp);
          gemm(tmp, rt, inv_i);
          invm = rec[14];
          const V3 com = ld3(rec) + scale(ld3(rec + 3), dt);  // position + (t - t0) velocity (:140)
          r = pc - com;
          double* v = A.vel + 6 * (size_t)b;
          st3(v, ld3(rec + 3));
          st3(v + 3, ld3(rec + 10));
        }
        st3(arm + 3 * s, r);
#pragma unroll
        for (int q = 0; q < 9; ++q) arm[6 + 9 * s + q] = inv_i[q];
        arm[24 + s] = invm;
      }
      arm[26] = add(mobility(arm[24], ld3(arm), arm + 6, nrm), mobility(arm[25], ld3(arm + 3), arm + 15, nrm));
    }
    __syncwarp();
    for (int k = lane; k < n; k += 32) {
      const int64_t c = c0 + k;
      double* arm = A.arm + (size_t)c * kArm;
      const V3 nrm = ld3(A.normal + 3 * c);
      const double vn0 = dot_blas(rel_vel(A, A.side[2 * c], A.side[2 * c + 1], ld3(arm), ld3(arm + 3)), nrm);
      arm[27] = mul(-A.restitution, 0.0 < vn0 ? 0.0 : vn0);  // -restitution * min(vn0, 0)
      A.lam[c] = 0.0;
      st3(A.fric + 3 * c, V3{0.0, 0.0, 0.0});
    }
    // ---- colour classes (:58-78), greedy in contact order on lane 0; a
    // body's classes below 64 are a bitset, higher ones are found by a scan
    for (int k = lane; k < n; k += 32) {
      const int64_t c = c0 + k;
      for (int s = 0; s < 2; ++s) {
        const int b = A.side[2 * c + s];
        if (b >= 0) A.cls[b] = 0ull;
      }
    }
    __syncwarp();
    int n_classes = 0;
    if (lane == 0) {
      for (int k = 0; k < n; ++k) {
        const int64_t c = c0 + k;
        const int ba = A.side[2 * c], bb = A.side[2 * c + 1];
        const unsigned long long taken = (ba >= 0 ? A.cls[ba] : 0ull) | (bb >= 0 ? A.cls[bb] : 0ull);
        int cl;
        if (taken != ~0ull) {
          cl = lowest_zero(taken);
        } else {  // rare: classes >= 64, scan the earlier contacts sharing a body
          cl = 64;
          bool again = true;
          while (again) {
            again = false;
            for (int j = 0; j < k; ++j) {
              const int64_t e = c0 + j;
              if (A.color[e] != cl) continue;
              const int ea = A.side[2 * e], eb = A.side[2 * e + 1];
              if ((ba >= 0 && (ea == ba || eb == ba)) || (bb >= 0 && (ea == bb || eb == bb))) {
                ++cl;
                again = true;
                break;
              }
            }
          }
        }
        A.color[c] = cl;
        if (cl < 64) {
          if (ba >= 0) A.cls[ba] |= 1ull << cl;
          if (bb >= 0) A.cls[bb] |= 1ull << cl;
        }
        n_classes = max(n_classes, cl + 1);
      }
      // contacts by class (counting sort), class segments
      int32_t* seg = A.class_off + c0 + p;  // n_classes + 1 entries fit: n_classes <= n
      for (int q = 0; q <= n_classes; ++q) seg[q] = 0;
      for (int k = 0; k < n; ++k) ++seg[A.color[c0 + k] + 1];
      for (int q = 0; q < n_classes; ++q) seg[q + 1] += seg[q];
      for (int k = 0; k < n; ++k) A.order[c0 + seg[A.color[c0 + k]]++] = k;
      for (int q = n_classes; q > 0; --q) seg[q] = seg[q - 1];
      seg[0] = 0;
    }
    n_classes = __shfl_sync(0xffffffffu, n_classes, 0);
    __syncwarp();
    const int32_t* seg = A.class_off + c0 + p;
    // ---- sequential-impulse sweeps (:157-190)
    const double rp = mul(A.relaxation, A.penalty);
    int iterations = 0;
    bool conv = false;
    while (iterations < A.max_iterations && !conv) {
      ++iterations;
      double worst = 0.0;
      for (int q = 0; q < n_classes; ++q) {
        const int s0 = seg[q], s1 = seg[q + 1];
        for (int k = s0 + lane; k < s1; k += 32) {
          const int64_t c = c0 + A.order[c0 + k];
          const double* arm = A.arm + (size_t)c * kArm;
          const int ia = A.side[2 * c], ib = A.side[2 * c + 1];
          const V3 nrm = ld3(A.normal + 3 * c);
          const V3 ra = ld3(arm), rb = ld3(arm + 3);
          V3 v_rel = rel_vel(A, ia, ib, ra, rb);
          const double d_lam = dv(mul(rp, sub(arm[27], dot_blas(v_rel, nrm))), arm[26]);
          const double lam0 = A.lam[c];
          double new_lam = add(lam0, d_lam);
          if (0.0 > new_lam) new_lam = 0.0;  // max(lam + d_lam, 0.0)
          V3 applied = scale(nrm, sub(new_lam, lam0));
          A.lam[c] = new_lam;
          apply_imp(A, ia, ib, arm, applied);
          worst = fmax(worst, measure(ia, ib, arm, applied));
          if (A.friction > 0.0 && new_lam > 0.0) {
            v_rel = rel_vel(A, ia, ib, ra, rb);
            const V3 vt = v_rel - scale(nrm, dot_blas(v_rel, nrm));
            const double speed = norm_blas(vt);
            if (speed > 1e-12) {
              const V3 t_dir{dv(vt.x, speed), dv(vt.y, speed), dv(vt.z, speed)};
              const double k_t = add(mobility(arm[24], ra, arm + 6, t_dir), mobility(arm[25], rb, arm + 15, t_dir));
              const V3 f0 = ld3(A.fric + 3 * c);
              V3 target = f0 - scale(t_dir, dv(mul(A.relaxation, speed), k_t));
              const double cap = mul(A.friction, new_lam);
              const double sc = norm_blas(target);
              if (sc > cap) target = scale(target, dv(cap, sc));
              applied = target - f0;
              st3(A.fric + 3 * c, target);
              apply_imp(A, ia, ib, arm, applied);
              worst = fmax(worst, measure(ia, ib, arm, applied));
            }
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
      conv = worst < A.threshold;
    }
    // ---- outputs
    for (int k = lane; k < n; k += 32) {
      const int64_t c = c0 + k;
      for (int s = 0; s < 2; ++s) {
        const int b = A.side[2 * c + s];
        if (b < 0) continue;
        const double* v = A.vel + 6 * (size_t)b;
        st3(A.out_vel + 3 * (size_t)b, ld3(v));
        st3(A.out_ang + 3 * (size_t)b, ld3(v + 3));
        A.touched[b] = 1;
      }
    }
    if (lane == 0) {
      A.iterations[p] = iterations;
      A.converged[p] = conv ? 1 : 0;
    }
    __syncwarp();
  }
}

struct IntegrateArgs {
  const double* body;
  int32_t n_problems;
  const int64_t* member_off;
  const int32_t* member;
  const double* t_new;
  const int64_t* off;
  const int32_t* side;
  const int64_t* id;
  const double* normal;
  const double* t;
  const double* depth;
  const double* vel;
  const double* ang;
  const int32_t* touched;
  double beta;
  int32_t separate;
  const double* new_in;  // separation only (apply_separation alone): the members' new snapshots
  double* first;     // scratch: first contact time per body
  int32_t* sep;      // scratch: positive-depth contacts of a problem, sorted
  double* out;       // n_bodies x 14
};

__device__ __forceinline__ void atomic_min_double(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (v < __longlong_as_double((long long)old)) {
    const unsigned long long prev = atomicCAS(a, old, (unsigned long long)__double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

__global__ void k_integrate(IntegrateArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < A.n_problems; p += nw) {
    const int64_t m0 = A.member_off[p], m1 = A.member_off[p + 1];
    const int64_t c0 = A.off[p], c1 = A.off[p + 1];
    for (int64_t k = m0 + lane; k < m1; k += 32) A.first[A.member[k]] = CUDART_INF;
    __syncwarp();
    for (int64_t c = c0 + lane; c < c1; c += 32)  // first_touch (:236-241): a min, order-free
      for (int s = 0; s < 2; ++s) {
        const int b = A.side[2 * c + s];
        if (b >= 0) atomic_min_double(A.first + b, A.t[c]);
      }
    __syncwarp();
    const double t_new = A.t_new[p];
    for (int64_t k = m0 + lane; k < m1; k += 32) {  // (:242-253)
      const int b = A.member[k];
      const double* rec = A.body + (size_t)b * kBody;
      const double tc = A.first[b];
      double* o = A.out + (size_t)b * 14;
      V3 pos, vel = ld3(rec + 3), om = ld3(rec + 10);
      double q[4], t;
      if (A.new_in != nullptr) {  // separation only: start from the given new snapshots
        const double* s = A.new_in + (size_t)b * 14;
        for (int i = 0; i < 14; ++i) o[i] = s[i];
        continue;
      }
      if (tc == CUDART_INF || A.vel == nullptr || !A.touched[b]) {
        const double dt = sub(t_new, rec[13]);
        flight(rec, dt, &pos, q);
        t = add(rec[13], dt);
      } else {
        const double dt1 = sub(tc, rec[13]);
        V3 p1;
        double q1[4];
        flight(rec, dt1, &p1, q1);
        const double t1 = add(rec[13], dt1);
        vel = ld3(A.vel + 3 * (size_t)b);
        om = ld3(A.ang + 3 * (size_t)b);
        const double dt2 = sub(t_new, t1);
        pos = p1 + scale(vel, dt2);
        advance(q1, om, dt2, q);
        t = add(t1, dt2);
      }
      st3(o, pos);
      st3(o + 3, vel);
      for (int i = 0; i < 4; ++i) o[6 + i] = q[i];
      st3(o + 10, om);
      o[13] = t;
    }
    __syncwarp();
    if (lane == 0 && A.separate) {  // apply_separation (:256-285): groups in sorted (id_a, id_b) order
      int m = 0;
      int32_t* idx = A.sep + c0;
      for (int64_t c = c0; c < c1; ++c) {
        if (!(A.depth[c] > 0.0)) continue;
        // stable insertion by the group key
        const int64_t ka = A.id[2 * c], kb = A.id[2 * c + 1];
        int j = m++;
        while (j > 0) {
          const int64_t e = c0 + idx[j - 1];
          const int64_t ea = A.id[2 * e], eb = A.id[2 * e + 1];
          if (ea < ka || (ea == ka && eb <= kb)) break;
          idx[j] = idx[j - 1];
          --j;
        }
        idx[j] = (int32_t)(c - c0);
      }
      int g = 0;
      while (g < m) {
        const int64_t e0 = c0 + idx[g];
        const int64_t ka = A.id[2 * e0], kb = A.id[2 * e0 + 1];
        int h = g;
        V3 acc{0.0, 0.0, 0.0};
        while (h < m) {
          const int64_t e = c0 + idx[h];
          if (A.id[2 * e] != ka || A.id[2 * e + 1] != kb) break;
          const V3 v = scale(ld3(A.normal + 3 * e), A.depth[e]);
          acc = h == g ? v : acc + v;  // np.mean(axis=0): rows summed in order
          ++h;
        }
        const int ia = A.side[2 * e0], ib = A.side[2 * e0 + 1];
        const double wa = ia >= 0 ? A.body[(size_t)ia * kBody + 14] : 0.0;
        const double wb = ib >= 0 ? A.body[(size_t)ib * kBody + 14] : 0.0;
        const double total = add(wa, wb);
        if (total != 0.0) {
          const double cnt = (double)(h - g);
          const V3 push = scale(V3{dv(acc.x, cnt), dv(acc.y, cnt), dv(acc.z, cnt)}, A.beta);
          if (ia >= 0) {
            double* o = A.out + (size_t)ia * 14;
            st3(o, ld3(o) + scale(push, dv(wa, total)));
          }
          if (ib >= 0) {
            double* o = A.out + (size_t)ib * 14;
            st3(o, ld3(o) - scale(push, dv(wb, total)));
          }
        }
        g = h;
      }
    }
    __syncwarp();
  }
}

template <typename T>
static int wsget(ltsg_workspace* ws, const char* name, int64_t count, T** out) {
  void* p = nullptr;
  LTSG_TRY(ws->get(name, (size_t)(count > 0 ? count : 1) * sizeof(T), &p));
  *out = (T*)p;
  return LTSG_OK;
}

static int warps_grid(int n_problems) {
  const int64_t blocks = ((int64_t)n_problems * 32 + 127) / 128;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16));
}

}  // namespace cs
}  // namespace ltsg

using namespace ltsg;
using namespace ltsg::cs;

extern "C" {

int ltsg_solve_impulses(const ltsg_solve_input* in, ltsg_solve_output* out, ltsg_workspace* ws, void* stream) {
  if (!in || !out || !ws || in->n_bodies < 0 || in->n_problems < 0 || in->n_contacts < 0 ||
      (in->n_contacts > 0 && (!in->side || !in->position || !in->normal || !in->t || !in->body)) ||
      !in->contact_offset || in->max_iterations < 1 || !out->iterations || !out->converged ||
      (in->n_contacts > 0 && (!out->normal_impulse || !out->friction_impulse || !out->color)) ||
      (in->n_bodies > 0 && (!out->velocity || !out->angular_velocity || !out->touched))) {
    set_error("ltsg_solve_impulses: bad arguments");
    return LTSG_EINVAL;
  }
  out->launches = 0;
  out->ms = 0.0;
  if (in->n_problems == 0) return LTSG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t e0 = ws->event(0), e1 = ws->event(1);
  LTSG_CUDA(cudaEventRecord(e0, st));
  SolveArgs A{};
  A.body = in->body;
  A.off = in->contact_offset;
  A.side = in->side;
  A.position = in->position;
  A.normal = in->normal;
  A.t = in->t;
  A.restitution = in->restitution;
  A.friction = in->friction;
  A.relaxation = in->relaxation;
  A.penalty = in->penalty;
  A.threshold = in->threshold;
  A.max_iterations = in->max_iterations;
  A.n_problems = in->n_problems;
  LTSG_TRY(wsget(ws, "cs_arm", in->n_contacts * kArm, &A.arm));
  LTSG_TRY(wsget(ws, "cs_vel", (int64_t)in->n_bodies * 6, &A.vel));
  LTSG_TRY(wsget(ws, "cs_cls", in->n_bodies, &A.cls));
  LTSG_TRY(wsget(ws, "cs_order", in->n_contacts, &A.order));
  LTSG_TRY(wsget(ws, "cs_seg", in->n_contacts + in->n_problems + 1, &A.class_off));
  A.out_vel = out->velocity;
  A.out_ang = out->angular_velocity;
  A.touched = out->touched;
  A.lam = out->normal_impulse;
  A.fric = out->friction_impulse;
  A.color = out->color;
  A.iterations = out->iterations;
  A.converged = out->converged;
  if (in->n_bodies > 0) LTSG_CUDA(cudaMemsetAsync(out->touched, 0, sizeof(int32_t) * in->n_bodies, st));
  k_solve<<<warps_grid(in->n_problems), 128, 0, st>>>(A);
  LTSG_CHECK_LAUNCH();
  out->launches = 1;
  LTSG_CUDA(cudaEventRecord(e1, st));
  LTSG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  LTSG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  out->ms = (double)ms;
  return LTSG_OK;
}

int ltsg_integrate(const ltsg_integrate_input* in, double* new_state, ltsg_workspace* ws, void* stream) {
  if (!in || !ws || !new_state || in->n_bodies < 0 || in->n_problems < 0 || in->n_contacts < 0 ||
      !in->member_offset || !in->t_new || !in->contact_offset || (in->n_bodies > 0 && !in->body) ||
      (in->n_contacts > 0 && (!in->side || !in->id || !in->normal || !in->t || !in->depth)) ||
      (in->velocity && (!in->angular_velocity || !in->touched))) {
    set_error("ltsg_integrate: bad arguments");
    return LTSG_EINVAL;
  }
  if (in->n_problems == 0) return LTSG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  IntegrateArgs A{};
  A.body = in->body;
  A.n_problems = in->n_problems;
  A.member_off = in->member_offset;
  A.member = in->member;
  A.t_new = in->t_new;
  A.off = in->contact_offset;
  A.side = in->side;
  A.id = in->id;
  A.normal = in->normal;
  A.t = in->t;
  A.depth = in->depth;
  A.vel = in->velocity;
  A.ang = in->angular_velocity;
  A.touched = in->touched;
  A.beta = in->beta;
  A.new_in = in->new_state_in;
  A.separate = in->separate;
  A.out = new_state;
  LTSG_TRY(wsget(ws, "cs_first", in->n_bodies, &A.first));
  LTSG_TRY(wsget(ws, "cs_sep", in->n_contacts, &A.sep));
  k_integrate<<<warps_grid(in->n_problems), 128, 0, st>>>(A);
  LTSG_CHECK_LAUNCH();
  return LTSG_OK;
}

}  // extern "C"
