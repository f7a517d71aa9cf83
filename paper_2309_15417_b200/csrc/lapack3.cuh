// The plane-fit basis of ltsdem.surrogate._fit_parent_triangle
// (surrogate.py:49-68): `np.linalg.svd(rel, full_matrices=False)` of an
// m x 3 matrix (m = 3, 6, 9 or 12 points), restated so that V^T comes out
// bit-identical to what numpy computes on the build host.
//
// numpy 2.3 hands the matrix to LAPACK dgesdd (JOBZ='S') from its bundled
// OpenBLAS 0.3.30 (SkylakeX kernels on the build and GPU hosts).  For m x 3
// that routine runs
//   m >= 5 (MNTHR = int(3*11/6)):  dgeqr2 -> R = triu -> dgebd2(R)
//   m <  5:                        dgebd2(A)
//   then dbdsdc('U','I') = dlasdq -> dbdsqr, dlasdq's and dbdsdc's sorts,
//   and dormbr('P','R','T') = dorml2 applying the right reflectors to VT.
// The LAPACK Fortran is compiled without FMA (separately rounded IEEE
// operations, which -fmad=false plus the __d*_rn helpers give here).  The
// BLAS calls inside it are OpenBLAS kernels with their own summation orders,
// pinned by probing the library (tools/blas_probe.py, oracle/lapack_svd.py):
//   dnrm2     x87 extended precision: four 64-bit-mantissa accumulators,
//             fsqrt, one rounding to double (emulated exactly with integers)
//   dgemv_t   SSE2 4x2 / 4x1 kernels over the rows m & ~3, then the scalar
//             tail rows with the compiler's FMA contraction
//   dgemv_n   (m <= 3 rows) one FMA chain per row over the columns
//   dger      a[i,j] = fma(alpha*y[j], x[i], a[i,j])
//   drot      x' = fma(c, x, s*y), y' = fma(c, y, -(s*x))
// oracle/lapack_svd.py is the Python statement of the same algorithm; it and
// this file agree bit for bit with numpy on random, degenerate (tied and
// zero singular values, exact zeros) and surrogate-tree matrices.
#pragma once

#include "geom.cuh"

namespace ltsg {
namespace lapack {

// ---------------------------------------------------------------- x87 dnrm2

struct X80 {  // value = m * 2^e; m == 0 or bit 63 of m set
  unsigned long long m;
  int e;
};

// round the 128-bit integer (hi:lo) * 2^e (plus a sticky tail) to 64 bits, RNE
__device__ inline X80 x80_round(unsigned long long hi, unsigned long long lo, int e, bool sticky) {
  if (hi == 0 && lo == 0) return X80{0ull, 0};
  const int lz = hi ? __clzll((long long)hi) : 64 + __clzll((long long)lo);
  if (lz >= 64) {
    hi = lo << (lz - 64);
    lo = 0;
  } else if (lz > 0) {
    hi = (hi << lz) | (lo >> (64 - lz));
    lo <<= lz;
  }
  e -= lz;
  const bool rb = (lo >> 63) != 0;
  const bool st = ((lo << 1) != 0) || sticky;
  e += 64;
  if (rb && (st || (hi & 1ull))) {
    hi += 1ull;
    if (hi == 0) {
      hi = 1ull << 63;
      e += 1;
    }
  }
  return X80{hi, e};
}

__device__ inline X80 x80_square(double x) {  // fld x; fmul st, st
  if (x == 0.0) return X80{0ull, 0};
  int k;
  const double f = frexp(fabs(x), &k);  // |x| = f * 2^k, f in [0.5, 1)
  const unsigned long long M = (unsigned long long)ldexp(f, 53);
  const int E = k - 53;
  return x80_round(__umul64hi(M, M), M * M, 2 * E, false);
}

__device__ inline X80 x80_add(X80 a, X80 b) {  // faddp, both operands >= 0
  if (a.m == 0) return b;
  if (b.m == 0) return a;
  if (a.e < b.e) {
    X80 t = a;
    a = b;
    b = t;
  }
  const int d = a.e - b.e;
  unsigned long long ah = a.m, al = 0, bh = b.m, bl = 0;
  bool sticky = false;
  if (d >= 128) {
    sticky = true;
    bh = bl = 0;
  } else if (d >= 64) {
    const int s = d - 64;
    sticky = s > 0 && (bh << (64 - s)) != 0;
    bl = s > 0 ? (bh >> s) : bh;
    bh = 0;
  } else if (d > 0) {
    bl = bh << (64 - d);
    bh >>= d;
  }
  unsigned long long lo = al + bl;
  const unsigned long long c0 = lo < al ? 1ull : 0ull;
  const unsigned long long s1 = ah + bh;
  unsigned long long hi = s1 + c0;
  const bool carry = s1 < ah || hi < s1;
  int e = a.e - 64;
  if (carry) {  // shift the 129-bit sum right by one
    sticky = sticky || (lo & 1ull);
    lo = (lo >> 1) | (hi << 63);
    hi = (hi >> 1) | (1ull << 63);
    e += 1;
  }
  return x80_round(hi, lo, e, sticky);
}

__device__ inline X80 x80_sqrt(X80 a) {  // fsqrt
  if (a.m == 0) return a;
  // N = m * 2^s in [2^126, 2^128) with (e - s) even; sqrt = sqrt(N) * 2^((e-s)/2)
  const int s = ((a.e - 64) & 1) ? 63 : 64;
  const unsigned long long nh = s == 64 ? a.m : (a.m >> 1);
  const unsigned long long nl = s == 64 ? 0ull : (a.m << 63);
  const double nd = ldexp((double)nh, 64) + (double)nl;
  double r0 = sqrt(nd);
  unsigned long long R = r0 >= 18446744073709549568.0 ? 0xFFFFFFFFFFFFF800ull : (unsigned long long)r0;
  if (R < (1ull << 63)) R = 1ull << 63;
  // integer correction: R = floor(sqrt(N))
  for (int it = 0; it < 64; ++it) {
    const unsigned long long qh = __umul64hi(R, R), ql = R * R;
    const bool gt = qh > nh || (qh == nh && ql > nl);
    if (gt) {
      const unsigned long long dl = ql - nl, dh = qh - nh - (ql < nl ? 1ull : 0ull);
      const double dd = ldexp((double)dh, 64) + (double)dl;
      unsigned long long step = (unsigned long long)(dd / (2.0 * (double)R));
      if (step < 1) step = 1;
      R -= step;
      continue;
    }
    // R^2 <= N: is (R+1)^2 <= N ?  (R+1)^2 = R^2 + 2R + 1
    const unsigned long long dl = nl - ql, dh = nh - qh - (nl < ql ? 1ull : 0ull);  // N - R^2 >= 0
    // N - R^2 >= 2R + 1 ?
    const unsigned long long tl = 2ull * R + 1ull, th = (R >> 63);  // 2R+1 as 128-bit (R < 2^64)
    const bool ge = dh > th || (dh == th && dl >= tl);
    if (!ge) {
      // rounding: RN64(sqrt(N)) = R + 1 iff N - R^2 > R (ties are impossible)
      const bool up = dh > 0 || dl > R;
      int e = (a.e - s) / 2;
      if (up) {
        R += 1ull;
        if (R == 0) {
          R = 1ull << 63;
          e += 1;
        }
      }
      return X80{R, e};
    }
    const double dd = ldexp((double)dh, 64) + (double)dl;
    unsigned long long step = (unsigned long long)(dd / (2.0 * (double)R));
    if (step < 1) step = 1;
    R += step;
  }
  return X80{R, (a.e - s) / 2};  // not reached for finite input
}

__device__ inline double x80_to_double(X80 a) {  // fstpl
  if (a.m == 0) return 0.0;
  return ldexp(__ull2double_rn(a.m), a.e);
}

// OpenBLAS dnrm2_k (x87): four accumulators over blocks of 8, the tail into
// the first, then ((a2 + a0) + a1) + a3, fsqrt, store.
__device__ inline double dnrm2(const double* x, int n, int inc) {
  if (n <= 0) return 0.0;
  if (n == 1) return fabs(x[0]);
  X80 acc[4] = {{0ull, 0}, {0ull, 0}, {0ull, 0}, {0ull, 0}};
  const int nb = n & ~7;
  for (int i = 0; i < nb; i += 4)
    for (int k = 0; k < 4; ++k) acc[k] = x80_add(acc[k], x80_square(x[(i + k) * inc]));
  for (int i = nb; i < n; ++i) acc[0] = x80_add(acc[0], x80_square(x[i * inc]));
  X80 t = x80_add(acc[2], acc[0]);
  t = x80_add(t, acc[1]);
  t = x80_add(acc[3], t);
  return x80_to_double(x80_sqrt(t));
}

// ---------------------------------------------------------------- LAPACK scalars

constexpr double kEps = 1.1102230246251565e-16;    // dlamch('E') = 2^-53
constexpr double kSafmin = 2.2250738585072014e-308;  // dlamch('S')

__device__ __forceinline__ double fsign(double a, double b) { return copysign(fabs(a), b); }

__device__ inline double dlapy2(double x, double y) {
  const double xa = fabs(x), ya = fabs(y);
  const double w = fmax(xa, ya), z = fmin(xa, ya);
  if (z == 0.0) return w;
  const double q = dv(z, w);
  return mul(w, __dsqrt_rn(add(1.0, mul(q, q))));
}

// dlartg (LAPACK >= 3.10, la_xlartg)
__device__ inline void dlartg(double f, double g, double* c, double* s, double* r) {
  if (g == 0.0) {
    *c = 1.0;
    *s = 0.0;
    *r = f;
    return;
  }
  if (f == 0.0) {
    *c = 0.0;
    *s = fsign(1.0, g);
    *r = fabs(g);
    return;
  }
  const double f1 = fabs(f), g1 = fabs(g);
  const double rtmin = 1.4916681462400413e-154;  // sqrt(safmin)
  const double rtmax = 4.740375954054589e+153;   // sqrt(safmax / 2)
  if (f1 > rtmin && f1 < rtmax && g1 > rtmin && g1 < rtmax) {
    const double d = __dsqrt_rn(add(mul(f, f), mul(g, g)));
    *c = dv(f1, d);
    *r = fsign(d, f);
    *s = dv(g, *r);
  } else {
    const double u = fmin(1.0 / kSafmin, fmax(kSafmin, fmax(f1, g1)));
    const double fs = dv(f, u), gs = dv(g, u);
    const double d = __dsqrt_rn(add(mul(fs, fs), mul(gs, gs)));
    *c = dv(fabs(fs), d);
    const double rr = fsign(d, f);
    *s = dv(gs, rr);
    *r = mul(rr, u);
  }
}

__device__ inline void dlas2(double f, double g, double h, double* ssmin, double* ssmax) {
  const double fa = fabs(f), ga = fabs(g), ha = fabs(h);
  const double fhmn = fmin(fa, ha), fhmx = fmax(fa, ha);
  if (fhmn == 0.0) {
    *ssmin = 0.0;
    if (fhmx == 0.0) {
      *ssmax = ga;
    } else {
      const double q = dv(fmin(fhmx, ga), fmax(fhmx, ga));
      *ssmax = mul(fmax(fhmx, ga), __dsqrt_rn(add(1.0, mul(q, q))));
    }
  } else if (ga < fhmx) {
    const double as = add(1.0, dv(fhmn, fhmx));
    const double at = dv(sub(fhmx, fhmn), fhmx);
    const double q = dv(ga, fhmx);
    const double au = mul(q, q);
    const double c = dv(2.0, add(__dsqrt_rn(add(mul(as, as), au)), __dsqrt_rn(add(mul(at, at), au))));
    *ssmin = mul(fhmn, c);
    *ssmax = dv(fhmx, c);
  } else {
    const double au = dv(fhmx, ga);
    if (au == 0.0) {
      *ssmin = dv(mul(fhmn, fhmx), ga);
      *ssmax = ga;
    } else {
      const double as = add(1.0, dv(fhmn, fhmx));
      const double at = dv(sub(fhmx, fhmn), fhmx);
      const double p = mul(as, au), q = mul(at, au);
      const double c = dv(1.0, add(__dsqrt_rn(add(1.0, mul(p, p))), __dsqrt_rn(add(1.0, mul(q, q)))));
      double mn = mul(mul(fhmn, c), au);
      *ssmin = add(mn, mn);
      *ssmax = dv(ga, add(c, c));
    }
  }
}

__device__ inline void dlasv2(double f, double g, double h, double* ssmin, double* ssmax, double* snr,
                              double* csr, double* snl, double* csl) {
  double ft = f, fa = fabs(f), ht = h, ha = fabs(h);
  int pmax = 1;
  const bool swap = ha > fa;
  if (swap) {
    pmax = 3;
    double t = ft;
    ft = ht;
    ht = t;
    t = fa;
    fa = ha;
    ha = t;
  }
  const double gt = g, ga = fabs(g);
  double clt, crt, slt, srt, smin, smax;
  if (ga == 0.0) {
    smin = ha;
    smax = fa;
    clt = 1.0;
    crt = 1.0;
    slt = 0.0;
    srt = 0.0;
  } else {
    bool gasmal = true;
    if (ga > fa) {
      pmax = 2;
      if (dv(fa, ga) < kEps) {
        gasmal = false;
        smax = ga;
        smin = ha > 1.0 ? dv(fa, dv(ga, ha)) : mul(dv(fa, ga), ha);
        clt = 1.0;
        slt = dv(ht, gt);
        srt = 1.0;
        crt = dv(ft, gt);
      }
    }
    if (gasmal) {
      const double d = sub(fa, ha);
      double l = d == fa ? 1.0 : dv(d, fa);
      const double m = dv(gt, ft);
      double t = sub(2.0, l);
      const double mm = mul(m, m), tt = mul(t, t);
      const double s = __dsqrt_rn(add(tt, mm));
      const double r = l == 0.0 ? fabs(m) : __dsqrt_rn(add(mul(l, l), mm));
      const double a = mul(0.5, add(s, r));
      smin = dv(ha, a);
      smax = mul(fa, a);
      if (mm == 0.0) {
        if (l == 0.0)
          t = mul(fsign(2.0, ft), fsign(1.0, gt));
        else
          t = add(dv(gt, fsign(d, ft)), dv(m, t));
      } else {
        t = mul(add(dv(m, add(s, t)), dv(m, add(r, l))), add(1.0, a));
      }
      l = __dsqrt_rn(add(mul(t, t), 4.0));
      crt = dv(2.0, l);
      srt = dv(t, l);
      clt = dv(add(crt, mul(srt, m)), a);
      slt = dv(mul(dv(ht, ft), srt), a);
    }
  }
  if (swap) {
    *csl = srt;
    *snl = crt;
    *csr = slt;
    *snr = clt;
  } else {
    *csl = clt;
    *snl = slt;
    *csr = crt;
    *snr = srt;
  }
  double tsign;
  if (pmax == 1)
    tsign = mul(mul(fsign(1.0, *csr), fsign(1.0, *csl)), fsign(1.0, f));
  else if (pmax == 2)
    tsign = mul(mul(fsign(1.0, *snr), fsign(1.0, *csl)), fsign(1.0, g));
  else
    tsign = mul(mul(fsign(1.0, *snr), fsign(1.0, *snl)), fsign(1.0, h));
  *ssmax = fsign(smax, tsign);
  *ssmin = fsign(smin, mul(mul(tsign, fsign(1.0, f)), fsign(1.0, h)));
}

// ---------------------------------------------------------------- BLAS kernels (OpenBLAS models)

// A is column-major with leading dimension lda: A[i + j*lda]
__device__ inline double gemv_t_k4x1(const double* a, const double* x, int nb) {
  double a10 = 0.0, a11 = 0.0, a90 = 0.0, a91 = 0.0;
  int i = 0;
  if (nb & 2) {
    a10 = add(a10, mul(a[0], x[0]));
    a11 = add(a11, mul(a[1], x[1]));
    i = 2;
  }
  for (; i < nb; i += 4) {
    a10 = add(a10, mul(a[i], x[i]));
    a11 = add(a11, mul(a[i + 1], x[i + 1]));
    a90 = add(a90, mul(a[i + 2], x[i + 2]));
    a91 = add(a91, mul(a[i + 3], x[i + 3]));
  }
  return add(add(a10, a90), add(a11, a91));
}

__device__ inline double gemv_t_k4x2(const double* a, const double* x, int nb) {
  double c0 = 0.0, c1 = 0.0;
  for (int i = 0; i < nb; i += 2) {
    c0 = add(c0, mul(a[i], x[i]));
    c1 = add(c1, mul(a[i + 1], x[i + 1]));
  }
  return add(c0, c1);
}

// y(0:n) = A(0:m, 0:n)^T x, alpha 1, beta 0 (dgemv 'T')
__device__ inline void gemv_t(const double* A, int lda, int m, int n, const double* x, double* y) {
  const int m3 = m & 3, m1 = m - m3;
  for (int j = 0; j < n; ++j) y[j] = 0.0;
  if (m1) {
    int j = 0;
    for (; j + 2 <= n; j += 2) {
      y[j] = fma_(gemv_t_k4x2(A + j * lda, x, m1), 1.0, y[j]);
      y[j + 1] = fma_(gemv_t_k4x2(A + (j + 1) * lda, x, m1), 1.0, y[j + 1]);
    }
    if (j < n) y[j] = fma_(gemv_t_k4x1(A + j * lda, x, m1), 1.0, y[j]);
  }
  for (int j = 0; j < n; ++j) {
    const double* a = A + j * lda + m1;
    const double* xt = x + m1;
    if (m3 == 1)
      y[j] = fma_(a[0], xt[0], y[j]);
    else if (m3 == 2)
      y[j] = add(y[j], fma_(a[0], xt[0], mul(a[1], xt[1])));
    else if (m3 == 3)
      y[j] = add(y[j], fma_(a[2], xt[2], fma_(a[0], xt[0], mul(a[1], xt[1]))));
  }
}

// y(0:m) = A(0:m, 0:n) x for m <= 3 (dgemv 'N' tail path)
__device__ inline void gemv_n(const double* A, int lda, int m, int n, const double* x, double* y) {
  double t[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) t[i] = fma_(A[i + j * lda], x[j], t[i]);
  for (int i = 0; i < m; ++i) y[i] = fma_(1.0, t[i], 0.0);
}

// A += alpha x y^T (dger)
__device__ inline void ger(double* A, int lda, int m, int n, const double* x, const double* y, double alpha) {
  for (int j = 0; j < n; ++j) {
    const double tmp = mul(alpha, y[j]);
    for (int i = 0; i < m; ++i) A[i + j * lda] = fma_(tmp, x[i], A[i + j * lda]);
  }
}

// ---------------------------------------------------------------- LAPACK routines

// dlarfg(n, alpha, x(incx)): returns tau, overwrites alpha with beta and x with v(2:n)
__device__ inline double dlarfg(int n, double* alpha, double* x, int incx) {
  if (n <= 1) return 0.0;
  const double xnorm = dnrm2(x, n - 1, incx);
  if (xnorm == 0.0) return 0.0;
  const double beta = -fsign(dlapy2(*alpha, xnorm), *alpha);
  const double tau = dv(sub(beta, *alpha), beta);
  const double sc = dv(1.0, sub(*alpha, beta));
  for (int i = 0; i < n - 1; ++i) x[i * incx] = mul(x[i * incx], sc);
  *alpha = beta;
  return tau;
}

__device__ inline int iladlc(int m, int n, const double* C, int ldc) {
  if (n == 0) return 0;
  if (C[(n - 1) * ldc] != 0.0 || C[(m - 1) + (n - 1) * ldc] != 0.0) return n;
  for (int j = n - 1; j >= 0; --j)
    for (int i = 0; i < m; ++i)
      if (C[i + j * ldc] != 0.0) return j + 1;
  return 0;
}

__device__ inline int iladlr(int m, int n, const double* C, int ldc) {
  if (m == 0) return 0;
  if (C[m - 1] != 0.0 || C[(m - 1) + (n - 1) * ldc] != 0.0) return m;
  int r = 0;
  for (int j = 0; j < n; ++j) {
    int i = m;
    while (i >= 1 && C[(i - 1) + j * ldc] == 0.0) --i;
    r = r > i ? r : i;
  }
  return r;
}

// dlarf('L'): C(m x n) := (I - tau v v^T) C, v contiguous (v[0] = 1 stored by the caller)
__device__ inline void dlarf_left(const double* v, double tau, double* C, int ldc, int m, int n) {
  if (tau == 0.0) return;
  int lv = m;
  while (lv > 0 && v[lv - 1] == 0.0) --lv;
  if (lv == 0) return;
  const int lc = iladlc(lv, n, C, ldc);
  if (lc == 0) return;
  double w[3];
  gemv_t(C, ldc, lv, lc, v, w);
  ger(C, ldc, lv, lc, v, w, -tau);
}

// dlarf('R'): C(m x n) := C (I - tau v v^T), m <= 3, v contiguous
__device__ inline void dlarf_right(const double* v, double tau, double* C, int ldc, int m, int n) {
  if (tau == 0.0) return;
  int lv = n;
  while (lv > 0 && v[lv - 1] == 0.0) --lv;
  if (lv == 0) return;
  const int lc = iladlr(m, lv, C, ldc);
  if (lc == 0) return;
  double w[3];
  gemv_n(C, ldc, lc, lv, v, w);
  ger(C, ldc, lc, lv, w, v, -tau);
}

// DLASR('L','V','F'|'B') on rows r0..r0+k of the 3x3 column-major VT
__device__ inline void dlasr_l(double* VT, int r0, int k, const double* c, const double* s, bool forward) {
  for (int jj = 0; jj < k - 1; ++jj) {
    const int j = forward ? jj : k - 2 - jj;
    const double ct = c[j], st = s[j];
    if (ct != 1.0 || st != 0.0) {
      const int ra = r0 + j, rb = r0 + j + 1;
      for (int i = 0; i < 3; ++i) {
        const double temp = VT[rb + 3 * i];
        VT[rb + 3 * i] = sub(mul(ct, temp), mul(st, VT[ra + 3 * i]));
        VT[ra + 3 * i] = add(mul(st, temp), mul(ct, VT[ra + 3 * i]));
      }
    }
  }
}

__device__ __forceinline__ void swap_rows(double* VT, int a, int b) {
  for (int i = 0; i < 3; ++i) {
    const double t = VT[a + 3 * i];
    VT[a + 3 * i] = VT[b + 3 * i];
    VT[b + 3 * i] = t;
  }
}

// dbdsqr('U', n = 3, ncvt = 3, nru = 0, ncc = 0) with VT column-major 3x3;
// d[3], e[2] (1-based indices of the Fortran are written as [i-1]).
// Returns false if it did not converge (LAPACK would report INFO > 0).
__device__ inline bool dbdsqr3(double* d, double* e, double* VT) {
  const int n = 3;
  const double tolmul = 98.70149282610821;  // max(10, min(100, eps**(-0.125)))
  const double tol = mul(tolmul, kEps);
  double smax = 0.0;
  for (int i = 0; i < n; ++i) smax = fmax(smax, fabs(d[i]));
  for (int i = 0; i < n - 1; ++i) smax = fmax(smax, fabs(e[i]));
  double sminoa = fabs(d[0]);
  if (sminoa != 0.0) {
    double mu = sminoa;
    for (int i = 1; i < n; ++i) {
      mu = mul(fabs(d[i]), dv(mu, add(mu, fabs(e[i - 1]))));
      sminoa = fmin(sminoa, mu);
      if (sminoa == 0.0) break;
    }
  }
  sminoa = dv(sminoa, __dsqrt_rn((double)n));
  const double thresh = fmax(mul(tol, sminoa), mul(6.0, mul((double)n, mul((double)n, kSafmin))));
  const int maxit = 6 * n * n;  // MAXITDIVN * N iterations of N: generous bound
  int iter = 0;
  int idir = 0, oldll = -1, oldm = -1;
  int m = n;
  double smin = 0.0;
  while (m > 1) {
    if (++iter > 64 * maxit) return false;
    smax = fabs(d[m - 1]);
    int ll = 0;
    bool split = false;
    for (int lll = 1; lll <= m - 1; ++lll) {
      const int l1 = m - lll;
      const double abss = fabs(d[l1 - 1]), abse = fabs(e[l1 - 1]);
      if (abse <= thresh) {
        e[l1 - 1] = 0.0;
        ll = l1;
        split = true;
        break;
      }
      smax = fmax(smax, fmax(abss, abse));
    }
    if (split && ll == m - 1) {
      m -= 1;
      continue;
    }
    if (!split) ll = 0;
    ll += 1;
    if (ll == m - 1) {
      double sigmn, sigmx, sinr, cosr, sinl, cosl;
      dlasv2(d[m - 2], e[m - 2], d[m - 1], &sigmn, &sigmx, &sinr, &cosr, &sinl, &cosl);
      d[m - 2] = sigmx;
      e[m - 2] = 0.0;
      d[m - 1] = sigmn;
      const int r0 = m - 2, r1 = m - 1;
      for (int i = 0; i < 3; ++i) {  // drot
        const double x = VT[r0 + 3 * i], y = VT[r1 + 3 * i];
        VT[r0 + 3 * i] = fma_(cosr, x, mul(sinr, y));
        VT[r1 + 3 * i] = fma_(cosr, y, -mul(sinr, x));
      }
      m -= 2;
      continue;
    }
    if (ll > oldm || m < oldll) idir = fabs(d[ll - 1]) >= fabs(d[m - 1]) ? 1 : 2;
    if (idir == 1) {
      if (fabs(e[m - 2]) <= mul(fabs(tol), fabs(d[m - 1]))) {
        e[m - 2] = 0.0;
        continue;
      }
      double mu = fabs(d[ll - 1]);
      smin = mu;
      bool conv = false;
      for (int lll = ll; lll <= m - 1; ++lll) {
        if (fabs(e[lll - 1]) <= mul(tol, mu)) {
          e[lll - 1] = 0.0;
          conv = true;
          break;
        }
        mu = mul(fabs(d[lll]), dv(mu, add(mu, fabs(e[lll - 1]))));
        smin = fmin(smin, mu);
      }
      if (conv) continue;
    } else {
      if (fabs(e[ll - 1]) <= mul(fabs(tol), fabs(d[ll - 1]))) {
        e[ll - 1] = 0.0;
        continue;
      }
      double mu = fabs(d[m - 1]);
      smin = mu;
      bool conv = false;
      for (int lll = m - 1; lll >= ll; --lll) {
        if (fabs(e[lll - 1]) <= mul(tol, mu)) {
          e[lll - 1] = 0.0;
          conv = true;
          break;
        }
        mu = mul(fabs(d[lll - 1]), dv(mu, add(mu, fabs(e[lll - 1]))));
        smin = fmin(smin, mu);
      }
      if (conv) continue;
    }
    oldll = ll;
    oldm = m;
    double shift;
    if (mul(mul((double)n, tol), dv(smin, smax)) <= fmax(kEps, mul(0.01, tol))) {
      shift = 0.0;
    } else {
      double sll, r;
      if (idir == 1) {
        sll = fabs(d[ll - 1]);
        dlas2(d[m - 2], e[m - 2], d[m - 1], &shift, &r);
      } else {
        sll = fabs(d[m - 1]);
        dlas2(d[ll - 1], e[ll - 1], d[ll], &shift, &r);
      }
      if (sll > 0.0) {
        const double q = dv(shift, sll);
        if (mul(q, q) < kEps) shift = 0.0;
      }
    }
    const int k = m - ll;  // rotations
    double c1[3], s1[3], c2[3], s2[3];
    if (shift == 0.0) {
      if (idir == 1) {
        double cs = 1.0, sn = 0.0, oldcs = 1.0, oldsn = 0.0, r;
        for (int i = ll; i <= m - 1; ++i) {
          dlartg(mul(d[i - 1], cs), e[i - 1], &cs, &sn, &r);
          if (i > ll) e[i - 2] = mul(oldsn, r);
          double dnew;
          dlartg(mul(oldcs, r), mul(d[i], sn), &oldcs, &oldsn, &dnew);
          d[i - 1] = dnew;
          c1[i - ll] = cs;
          s1[i - ll] = sn;
          c2[i - ll] = oldcs;
          s2[i - ll] = oldsn;
        }
        const double h = mul(d[m - 1], cs);
        d[m - 1] = mul(h, oldcs);
        e[m - 2] = mul(h, oldsn);
        dlasr_l(VT, ll - 1, k + 1, c1, s1, true);
        if (fabs(e[m - 2]) <= thresh) e[m - 2] = 0.0;
      } else {
        double cs = 1.0, sn = 0.0, oldcs = 1.0, oldsn = 0.0, r;
        for (int i = m; i >= ll + 1; --i) {
          dlartg(mul(d[i - 1], cs), e[i - 2], &cs, &sn, &r);
          if (i < m) e[i - 1] = mul(oldsn, r);
          double dnew;
          dlartg(mul(oldcs, r), mul(d[i - 2], sn), &oldcs, &oldsn, &dnew);
          d[i - 1] = dnew;
          const int j = i - ll - 1;
          c1[j] = cs;
          s1[j] = -sn;
          c2[j] = oldcs;
          s2[j] = -oldsn;
        }
        const double h = mul(d[ll - 1], cs);
        d[ll - 1] = mul(h, oldcs);
        e[ll - 1] = mul(h, oldsn);
        dlasr_l(VT, ll - 1, k + 1, c2, s2, false);
        if (fabs(e[ll - 1]) <= thresh) e[ll - 1] = 0.0;
      }
    } else {
      if (idir == 1) {
        double f = mul(sub(fabs(d[ll - 1]), shift), add(fsign(1.0, d[ll - 1]), dv(shift, d[ll - 1])));
        double g = e[ll - 1];
        for (int i = ll; i <= m - 1; ++i) {
          double cosr, sinr, cosl, sinl, r;
          dlartg(f, g, &cosr, &sinr, &r);
          if (i > ll) e[i - 2] = r;
          f = add(mul(cosr, d[i - 1]), mul(sinr, e[i - 1]));
          e[i - 1] = sub(mul(cosr, e[i - 1]), mul(sinr, d[i - 1]));
          g = mul(sinr, d[i]);
          d[i] = mul(cosr, d[i]);
          dlartg(f, g, &cosl, &sinl, &r);
          d[i - 1] = r;
          f = add(mul(cosl, e[i - 1]), mul(sinl, d[i]));
          d[i] = sub(mul(cosl, d[i]), mul(sinl, e[i - 1]));
          if (i < m - 1) {
            g = mul(sinl, e[i]);
            e[i] = mul(cosl, e[i]);
          }
          c1[i - ll] = cosr;
          s1[i - ll] = sinr;
          c2[i - ll] = cosl;
          s2[i - ll] = sinl;
        }
        e[m - 2] = f;
        dlasr_l(VT, ll - 1, k + 1, c1, s1, true);
        if (fabs(e[m - 2]) <= thresh) e[m - 2] = 0.0;
      } else {
        double f = mul(sub(fabs(d[m - 1]), shift), add(fsign(1.0, d[m - 1]), dv(shift, d[m - 1])));
        double g = e[m - 2];
        for (int i = m; i >= ll + 1; --i) {
          double cosr, sinr, cosl, sinl, r;
          dlartg(f, g, &cosr, &sinr, &r);
          if (i < m) e[i - 1] = r;
          f = add(mul(cosr, d[i - 1]), mul(sinr, e[i - 2]));
          e[i - 2] = sub(mul(cosr, e[i - 2]), mul(sinr, d[i - 1]));
          g = mul(sinr, d[i - 2]);
          d[i - 2] = mul(cosr, d[i - 2]);
          dlartg(f, g, &cosl, &sinl, &r);
          d[i - 1] = r;
          f = add(mul(cosl, e[i - 2]), mul(sinl, d[i - 2]));
          d[i - 2] = sub(mul(cosl, d[i - 2]), mul(sinl, e[i - 2]));
          if (i > ll + 1) {
            g = mul(sinl, e[i - 3]);
            e[i - 3] = mul(cosl, e[i - 3]);
          }
          const int j = i - ll - 1;
          c1[j] = cosr;
          s1[j] = -sinr;
          c2[j] = cosl;
          s2[j] = -sinl;
        }
        e[ll - 1] = f;
        if (fabs(e[ll - 1]) <= thresh) e[ll - 1] = 0.0;
        dlasr_l(VT, ll - 1, k + 1, c2, s2, false);
      }
    }
  }
  // make the singular values positive (dscal(-1) of the VT row)
  for (int i = 0; i < n; ++i)
    if (d[i] < 0.0) {
      d[i] = -d[i];
      for (int c = 0; c < 3; ++c) VT[i + 3 * c] = -VT[i + 3 * c];
    }
  // dbdsqr's sort: smallest to the end, `<=` (ties keep their order)
  for (int i = 0; i < n - 1; ++i) {
    int isub = 0;
    double sm = d[0];
    for (int j = 1; j < n - i; ++j)
      if (d[j] <= sm) {
        isub = j;
        sm = d[j];
      }
    if (isub != n - 1 - i) {
      d[isub] = d[n - 1 - i];
      d[n - 1 - i] = sm;
      swap_rows(VT, isub, n - 1 - i);
    }
  }
  // dlasdq's selection sort (smallest first, strict <), then dbdsdc's
  // (largest first, strict >): no-ops unless values tie exactly
  for (int i = 0; i < n; ++i) {
    int isub = i;
    double sm = d[i];
    for (int j = i + 1; j < n; ++j)
      if (d[j] < sm) {
        isub = j;
        sm = d[j];
      }
    if (isub != i) {
      d[isub] = d[i];
      d[i] = sm;
      swap_rows(VT, isub, i);
    }
  }
  for (int i = 0; i < n - 1; ++i) {
    int kk = i;
    double p = d[i];
    for (int j = i + 1; j < n; ++j)
      if (d[j] > p) {
        kk = j;
        p = d[j];
      }
    if (kk != i) {
      d[kk] = d[i];
      d[i] = p;
      swap_rows(VT, kk, i);
    }
  }
  return true;
}

constexpr int kLda = 24;  // rows of the point matrix: 3 x fanout, fanout <= 8

// V^T (3x3, column-major) of the m x 3 matrix A (column-major, lda = kLda,
// overwritten) as dgesdd(JOBZ='S') returns it.  m in 3..kLda.
__device__ inline bool svd_vt(double* A, int m, double* VT) {
  constexpr int lda = kLda;
  double R[9];  // 3x3 column-major, ld 3
  if (m >= 5) {
    for (int i = 0; i < 3; ++i) {  // dgeqr2
      double alpha = A[i + i * lda];
      const double tau = dlarfg(m - i, &alpha, &A[(i + 1) + i * lda], 1);
      A[i + i * lda] = alpha;
      if (i < 2) {
        const double aii = A[i + i * lda];
        A[i + i * lda] = 1.0;
        dlarf_left(&A[i + i * lda], tau, &A[i + (i + 1) * lda], lda, m - i, 2 - i);
        A[i + i * lda] = aii;
      }
    }
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) R[i + 3 * j] = i <= j ? A[i + j * lda] : 0.0;
  } else {
    if (m < 3) return false;  // never: groups hold whole triangles (m = 3k)
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) R[i + 3 * j] = A[i + j * lda];
  }
  // dgebd2 on the 3x3 R (ld 3)
  double d[3], e[2], taup[3];
  for (int i = 0; i < 3; ++i) {
    double alpha = R[i + 3 * i];
    const double tq = dlarfg(3 - i, &alpha, &R[(i + 1 < 3 ? i + 1 : 2) + 3 * i], 1);
    d[i] = alpha;
    R[i + 3 * i] = 1.0;
    if (i < 2) dlarf_left(&R[i + 3 * i], tq, &R[i + 3 * (i + 1)], 3, 3 - i, 2 - i);
    R[i + 3 * i] = d[i];
    if (i < 2) {
      double a2 = R[i + 3 * (i + 1)];
      const int nx = 2 - i;  // length of the row reflector
      const double tp = dlarfg(nx, &a2, &R[i + 3 * (i + 2 < 3 ? i + 2 : 2)], 3);
      e[i] = a2;
      taup[i] = tp;
      R[i + 3 * (i + 1)] = 1.0;
      double v[2] = {1.0, nx > 1 ? R[i + 3 * (i + 2)] : 0.0};
      dlarf_right(v, tp, &R[(i + 1) + 3 * (i + 1)], 3, 2 - i, nx);
      R[i + 3 * (i + 1)] = e[i];
    } else {
      taup[i] = 0.0;
    }
  }
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) VT[i + 3 * j] = i == j ? 1.0 : 0.0;
  if (!dbdsqr3(d, e, VT)) return false;
  // dormbr('P','R','T'): VT(:, 2:3) := VT(:, 2:3) H(1), v = [1, R(1,3)], tau = taup(1)
  const double v[2] = {1.0, R[0 + 3 * 2]};
  dlarf_right(v, taup[0], &VT[3], 3, 3, 2);
  return true;
}

}  // namespace lapack
}  // namespace ltsg
