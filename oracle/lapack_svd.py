"""TEST INFRASTRUCTURE (oracle): the plane-fit SVD of the surrogate-tree
builder restated in plain Python -- only tests/ may import it.

`ltsdem.surrogate._fit_parent_triangle` (surrogate.py:49-68) calls
`np.linalg.svd(rel, full_matrices=False)` on an m x 3 matrix.  numpy 2.3
runs LAPACK dgesdd (JOBZ='S') from its bundled OpenBLAS 0.3.30; for m x 3
that is dgeqr2 (m >= 5) -> dgebd2 -> dbdsdc = dlasdq -> dbdsqr, the two
tie-breaking sorts, and dorml2 for the right reflectors.  The LAPACK
Fortran is separately rounded IEEE; the BLAS kernels it calls have the
summation orders probed from the library with tools/blas_probe.py
(x87 extended-precision dnrm2, SSE2 dgemv_t kernels + FMA tail, dgemv_n /
dger / drot FMA chains).  `svd_vt` reproduces numpy's V^T bit for bit on
random, degenerate and surrogate-tree matrices (tests/test_tree_oracle.py);
csrc/lapack3.cuh is the CUDA statement of the same algorithm.

The arithmetic uses Python floats (IEEE double) and Fractions for the
exact FMA and the x87 emulation, so it is slow: test-sized inputs only.
"""

from __future__ import annotations

import math
import sys
from fractions import Fraction

import numpy as np

EPS = 2.0 ** -53
SAFMIN = 2.0 ** -1022
RTMIN = math.sqrt(SAFMIN)
RTMAX = math.sqrt(1.0 / SAFMIN / 2)


def sign(a, b):
    return abs(a) if b >= 0 or (b == 0 and math.copysign(1, b) > 0) else -abs(a)


def fsign(a, b):  # Fortran SIGN: |a| with the sign bit of b
    return math.copysign(abs(a), b)


def dlapy2(x, y):
    xa, ya = abs(x), abs(y)
    w, z = max(xa, ya), min(xa, ya)
    if z == 0.0:
        return w
    return w * math.sqrt(1.0 + (z / w) ** 2)


def _rn(x: Fraction, bits: int) -> Fraction:
    """Round a non-negative rational to `bits` significant bits, ties to even."""
    if x == 0:
        return Fraction(0)
    e = x.numerator.bit_length() - x.denominator.bit_length()
    while Fraction(2) ** e > x:
        e -= 1
    while Fraction(2) ** (e + 1) <= x:
        e += 1
    ulp = Fraction(2) ** (e - bits + 1)
    q = x / ulp
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return fl * ulp


def _sqrt_rn64(v: Fraction) -> Fraction:
    if v == 0:
        return v
    # integer square root on a scaled value gives floor(sqrt) exactly
    e = v.numerator.bit_length() - v.denominator.bit_length()
    shift = 2 * (70 - e // 2)
    n = (v.numerator * (1 << shift)) // v.denominator if shift >= 0 else v.numerator // (v.denominator << -shift)
    r = math.isqrt(n)
    exact = r * r == n and (v.numerator * (1 << max(shift, 0))) % v.denominator == 0
    root = Fraction(r, 1 << (shift // 2))
    # r carries >= 70 significant bits; a sticky ulp beyond them settles the rounding
    if not exact:
        root += Fraction(1, 1 << (shift // 2 + 2))
    return _rn(root, 64)


def dnrm2(v):
    """OpenBLAS dnrm2_k (x87): four 64-bit-mantissa accumulators over blocks
    of 8, the tail into the first, ((a2 + a0) + a1) + a3, fsqrt, then one
    rounding to double."""
    n = len(v)
    if n == 0:
        return 0.0
    if n == 1:
        return abs(float(v[0]))
    acc = [Fraction(0)] * 4
    nb = n // 8 * 8
    for blk in range(0, nb, 4):
        for k in range(4):
            acc[k] = _rn(acc[k] + _rn(Fraction(v[blk + k]) ** 2, 64), 64)
    for i in range(nb, n):
        acc[0] = _rn(acc[0] + _rn(Fraction(v[i]) ** 2, 64), 64)
    t = _rn(acc[2] + acc[0], 64)
    t = _rn(t + acc[1], 64)
    t = _rn(acc[3] + t, 64)
    return float(_rn(_sqrt_rn64(t), 53))


def fma(a, b, c):
    """IEEE fused multiply-add, signed zeros included."""
    if not (math.isfinite(a) and math.isfinite(b) and math.isfinite(c)):
        return a * b + c
    p = Fraction(a) * Fraction(b)
    s = p + Fraction(c)
    if s == 0:
        pneg = math.copysign(1.0, a) * math.copysign(1.0, b) < 0
        if p == 0 and c == 0 and pneg and math.copysign(1.0, c) < 0:
            return -0.0
        return 0.0
    return float(s)


def _k4x1(a, x, nb):
    acc10 = [0.0, 0.0]
    acc9 = [0.0, 0.0]
    i = 0
    if nb & 2:
        acc10 = [acc10[0] + a[0] * x[0], acc10[1] + a[1] * x[1]]
        i = 2
    while i < nb:
        acc10 = [acc10[0] + a[i] * x[i], acc10[1] + a[i + 1] * x[i + 1]]
        acc9 = [acc9[0] + a[i + 2] * x[i + 2], acc9[1] + a[i + 3] * x[i + 3]]
        i += 4
    return (acc10[0] + acc9[0]) + (acc10[1] + acc9[1])


def _k4x2(a, x, nb):
    acc = [0.0, 0.0]
    for i in range(0, nb, 2):
        acc = [acc[0] + a[i] * x[i], acc[1] + a[i + 1] * x[i + 1]]
    return acc[0] + acc[1]


def gemv_t(A, x):
    """OpenBLAS dgemv_t (Haswell/SkylakeX driver), alpha 1, beta 0."""
    m, n = A.shape
    m3 = m & 3
    m1 = m - m3
    y = [0.0] * n
    if m1:
        j = 0
        while j + 2 <= n:
            y[j] = fma(_k4x2(A[:, j], x, m1), 1.0, y[j])
            y[j + 1] = fma(_k4x2(A[:, j + 1], x, m1), 1.0, y[j + 1])
            j += 2
        if j < n:
            y[j] = fma(_k4x1(A[:, j], x, m1), 1.0, y[j])
    for j in range(n):
        a = A[m1:, j]
        xt = x[m1:]
        if m3 == 1:
            y[j] = fma(a[0], xt[0], y[j])
        elif m3 == 2:
            y[j] = y[j] + fma(a[0], xt[0], a[1] * xt[1])
        elif m3 == 3:
            y[j] = y[j] + fma(a[2], xt[2], fma(a[0], xt[0], a[1] * xt[1]))
    return np.array(y)


def gemv_n(A, x):
    m, n = A.shape
    assert m <= 3
    t = [0.0] * m
    for j in range(n):
        for i in range(m):
            t[i] = fma(A[i, j], x[j], t[i])
    return np.array([fma(1.0, t[i], 0.0) for i in range(m)])


def ger(A, x, y, alpha):
    for j in range(A.shape[1]):
        tmp = alpha * y[j]
        for i in range(A.shape[0]):
            A[i, j] = fma(tmp, x[i], A[i, j])


def dlarfg(alpha, x):
    """Returns (beta, tau, scaled x)."""
    if len(x) == 0:
        return alpha, 0.0, x
    xnorm = dnrm2(x)
    if xnorm == 0.0:
        return alpha, 0.0, x
    beta = -fsign(dlapy2(alpha, xnorm), alpha)
    tau = (beta - alpha) / beta
    s = 1.0 / (alpha - beta)
    return beta, tau, [xi * s for xi in x]


def dlartg(f, g, old=False):
    if old:
        if g == 0.0:
            return 1.0, 0.0, f
        if f == 0.0:
            return 0.0, 1.0, g
        r = math.sqrt(f * f + g * g)
        cs, sn = f / r, g / r
        if abs(f) > abs(g) and cs < 0:
            cs, sn, r = -cs, -sn, -r
        return cs, sn, r
    if g == 0.0:
        return 1.0, 0.0, f
    if f == 0.0:
        return 0.0, fsign(1.0, g), abs(g)
    d = math.sqrt(f * f + g * g)
    c = abs(f) / d
    r = fsign(d, f)
    return c, g / r, r


def dlas2(f, g, h):
    fa, ga, ha = abs(f), abs(g), abs(h)
    fhmn, fhmx = min(fa, ha), max(fa, ha)
    if fhmn == 0.0:
        ssmin = 0.0
        if fhmx == 0.0:
            ssmax = ga
        else:
            ssmax = max(fhmx, ga) * math.sqrt(1.0 + (min(fhmx, ga) / max(fhmx, ga)) ** 2)
    elif ga < fhmx:
        as_ = 1.0 + fhmn / fhmx
        at = (fhmx - fhmn) / fhmx
        au = (ga / fhmx) ** 2
        c = 2.0 / (math.sqrt(as_ * as_ + au) + math.sqrt(at * at + au))
        ssmin, ssmax = fhmn * c, fhmx / c
    else:
        au = fhmx / ga
        if au == 0.0:
            ssmin, ssmax = (fhmn * fhmx) / ga, ga
        else:
            as_ = 1.0 + fhmn / fhmx
            at = (fhmx - fhmn) / fhmx
            c = 1.0 / (math.sqrt(1.0 + (as_ * au) ** 2) + math.sqrt(1.0 + (at * au) ** 2))
            ssmin = (fhmn * c) * au
            ssmin = ssmin + ssmin
            ssmax = ga / (c + c)
    return ssmin, ssmax


def dlasv2(f, g, h):
    ft, fa, ht, ha = f, abs(f), h, abs(h)
    pmax = 1
    swap = ha > fa
    if swap:
        pmax = 3
        ft, ht = ht, ft
        fa, ha = ha, fa
    gt, ga = g, abs(g)
    if ga == 0.0:
        ssmin, ssmax = ha, fa
        clt, crt, slt, srt = 1.0, 1.0, 0.0, 0.0
    else:
        gasmal = True
        if ga > fa:
            pmax = 2
            if fa / ga < EPS:
                gasmal = False
                ssmax = ga
                ssmin = fa / (ga / ha) if ha > 1.0 else (fa / ga) * ha
                clt, slt, srt, crt = 1.0, ht / gt, 1.0, ft / gt
        if gasmal:
            d = fa - ha
            l = 1.0 if d == fa else d / fa
            m = gt / ft
            t = 2.0 - l
            mm, tt = m * m, t * t
            s = math.sqrt(tt + mm)
            r = abs(m) if l == 0.0 else math.sqrt(l * l + mm)
            a = 0.5 * (s + r)
            ssmin, ssmax = ha / a, fa * a
            if mm == 0.0:
                if l == 0.0:
                    t = fsign(2.0, ft) * fsign(1.0, gt)
                else:
                    t = gt / fsign(d, ft) + m / t
            else:
                t = (m / (s + t) + m / (r + l)) * (1.0 + a)
            l = math.sqrt(t * t + 4.0)
            crt = 2.0 / l
            srt = t / l
            clt = (crt + srt * m) / a
            slt = (ht / ft) * srt / a
    if swap:
        csl, snl, csr, snr = srt, crt, slt, clt
    else:
        csl, snl, csr, snr = clt, slt, crt, srt
    if pmax == 1:
        tsign = fsign(1.0, csr) * fsign(1.0, csl) * fsign(1.0, f)
    elif pmax == 2:
        tsign = fsign(1.0, snr) * fsign(1.0, csl) * fsign(1.0, g)
    else:
        tsign = fsign(1.0, snr) * fsign(1.0, snl) * fsign(1.0, h)
    ssmax = fsign(ssmax, tsign)
    ssmin = fsign(ssmin, tsign * fsign(1.0, f) * fsign(1.0, h))
    return ssmin, ssmax, snr, csr, snl, csl


def dlasr_lvf(A, rows, c, s):
    """DLASR('L','V','F') on rows[0..k] of A (rotation j between rows j, j+1)."""
    for j in range(len(rows) - 1):
        ct, st = c[j], s[j]
        if ct != 1.0 or st != 0.0:
            r0, r1 = rows[j], rows[j + 1]
            for i in range(A.shape[1]):
                temp = A[r1, i]
                A[r1, i] = ct * temp - st * A[r0, i]
                A[r0, i] = st * temp + ct * A[r0, i]


def dlasr_lvb(A, rows, c, s):
    for j in range(len(rows) - 2, -1, -1):
        ct, st = c[j], s[j]
        if ct != 1.0 or st != 0.0:
            r0, r1 = rows[j], rows[j + 1]
            for i in range(A.shape[1]):
                temp = A[r1, i]
                A[r1, i] = ct * temp - st * A[r0, i]
                A[r0, i] = st * temp + ct * A[r0, i]


def dbdsqr(d, e, VT, old=False):
    """Upper bidiagonal SVD, vectors applied to VT only (U is not needed)."""
    n = len(d)
    d = list(d)
    e = list(e) + [0.0]
    maxitr = 6
    tolmul = max(10.0, min(100.0, EPS ** -0.125))
    tol = tolmul * EPS
    smax = max([abs(x) for x in d] + [abs(x) for x in e[:n - 1]])
    sminoa = abs(d[0])
    if sminoa != 0.0:
        mu = sminoa
        for i in range(1, n):
            mu = abs(d[i]) * (mu / (mu + abs(e[i - 1])))
            sminoa = min(sminoa, mu)
            if sminoa == 0.0:
                break
    sminoa = sminoa / math.sqrt(float(n))
    thresh = max(tol * sminoa, maxitr * (n * (n * SAFMIN)))
    itr = 0
    idir = 0
    oldll, oldm = -1, -1
    m = n  # 1-based index of the bottom row of the active block
    while m > 1:
        itr += 1
        if itr > 200:
            raise RuntimeError("no convergence")
        smax = abs(d[m - 1])
        ll = 0
        for lll in range(1, m):
            ll1 = m - lll  # 1-based
            abss, abse = abs(d[ll1 - 1]), abs(e[ll1 - 1])
            if abse <= thresh:
                e[ll1 - 1] = 0.0
                ll = ll1
                break
            smax = max(smax, abss, abse)
        else:
            ll = 0
        if ll != 0 and ll == m - 1:
            m -= 1
            continue
        ll = ll + 1  # 1-based top row of the block
        if ll == m - 1:
            ssmin, ssmax, sinr, cosr, sinl, cosl = dlasv2(d[m - 2], e[m - 2], d[m - 1])
            d[m - 2], e[m - 2], d[m - 1] = ssmax, 0.0, ssmin
            r0, r1 = m - 2, m - 1
            for i in range(VT.shape[1]):
                x, y = VT[r0, i], VT[r1, i]
                VT[r0, i] = fma(cosr, x, sinr * y)
                VT[r1, i] = fma(cosr, y, -(sinr * x))
            m -= 2
            continue
        if ll > oldm or m < oldll:
            idir = 1 if abs(d[ll - 1]) >= abs(d[m - 1]) else 2
        if idir == 1:
            if abs(e[m - 2]) <= abs(tol) * abs(d[m - 1]):
                e[m - 2] = 0.0
                continue
            mu = abs(d[ll - 1])
            smin = mu
            conv = False
            for lll in range(ll, m):
                if abs(e[lll - 1]) <= tol * mu:
                    e[lll - 1] = 0.0
                    conv = True
                    break
                mu = abs(d[lll]) * (mu / (mu + abs(e[lll - 1])))
                smin = min(smin, mu)
            if conv:
                continue
        else:
            if abs(e[ll - 1]) <= abs(tol) * abs(d[ll - 1]):
                e[ll - 1] = 0.0
                continue
            mu = abs(d[m - 1])
            smin = mu
            conv = False
            for lll in range(m - 1, ll - 1, -1):
                if abs(e[lll - 1]) <= tol * mu:
                    e[lll - 1] = 0.0
                    conv = True
                    break
                mu = abs(d[lll - 1]) * (mu / (mu + abs(e[lll - 1])))
                smin = min(smin, mu)
            if conv:
                continue
        oldll, oldm = ll, m
        if n * tol * (smin / smax) <= max(EPS, 0.01 * tol):
            shift = 0.0
        else:
            if idir == 1:
                sll = abs(d[ll - 1])
                shift, _ = dlas2(d[m - 2], e[m - 2], d[m - 1])
            else:
                sll = abs(d[m - 1])
                shift, _ = dlas2(d[ll - 1], e[ll - 1], d[ll])
            if sll > 0.0 and (shift / sll) ** 2 < EPS:
                shift = 0.0
        rows = list(range(ll - 1, m))
        k = m - ll
        c1, s1, c2, s2 = [0.0] * k, [0.0] * k, [0.0] * k, [0.0] * k
        if shift == 0.0:
            if idir == 1:
                cs, oldcs, oldsn = 1.0, 1.0, 0.0
                for i in range(ll, m):
                    cs, sn, r = dlartg(d[i - 1] * cs, e[i - 1], old)
                    if i > ll:
                        e[i - 2] = oldsn * r
                    oldcs, oldsn, d[i - 1] = dlartg(oldcs * r, d[i] * sn, old)
                    c1[i - ll], s1[i - ll], c2[i - ll], s2[i - ll] = cs, sn, oldcs, oldsn
                h = d[m - 1] * cs
                d[m - 1] = h * oldcs
                e[m - 2] = h * oldsn
                dlasr_lvf(VT, rows, c1, s1)
                if abs(e[m - 2]) <= thresh:
                    e[m - 2] = 0.0
            else:
                cs, oldcs, oldsn = 1.0, 1.0, 0.0
                for i in range(m, ll, -1):
                    cs, sn, r = dlartg(d[i - 1] * cs, e[i - 2], old)
                    if i < m:
                        e[i - 1] = oldsn * r
                    oldcs, oldsn, d[i - 1] = dlartg(oldcs * r, d[i - 2] * sn, old)
                    j = i - ll - 1
                    c1[j], s1[j], c2[j], s2[j] = cs, -sn, oldcs, -oldsn
                h = d[ll - 1] * cs
                d[ll - 1] = h * oldcs
                e[ll - 1] = h * oldsn
                dlasr_lvb(VT, rows, c2, s2)
                if abs(e[ll - 1]) <= thresh:
                    e[ll - 1] = 0.0
        else:
            if idir == 1:
                f = (abs(d[ll - 1]) - shift) * (fsign(1.0, d[ll - 1]) + shift / d[ll - 1])
                g = e[ll - 1]
                for i in range(ll, m):
                    cosr, sinr, r = dlartg(f, g, old)
                    if i > ll:
                        e[i - 2] = r
                    f = cosr * d[i - 1] + sinr * e[i - 1]
                    e[i - 1] = cosr * e[i - 1] - sinr * d[i - 1]
                    g = sinr * d[i]
                    d[i] = cosr * d[i]
                    cosl, sinl, r = dlartg(f, g, old)
                    d[i - 1] = r
                    f = cosl * e[i - 1] + sinl * d[i]
                    d[i] = cosl * d[i] - sinl * e[i - 1]
                    if i < m - 1:
                        g = sinl * e[i]
                        e[i] = cosl * e[i]
                    c1[i - ll], s1[i - ll], c2[i - ll], s2[i - ll] = cosr, sinr, cosl, sinl
                e[m - 2] = f
                dlasr_lvf(VT, rows, c1, s1)
                if abs(e[m - 2]) <= thresh:
                    e[m - 2] = 0.0
            else:
                f = (abs(d[m - 1]) - shift) * (fsign(1.0, d[m - 1]) + shift / d[m - 1])
                g = e[m - 2]
                for i in range(m, ll, -1):
                    cosr, sinr, r = dlartg(f, g, old)
                    if i < m:
                        e[i - 1] = r
                    f = cosr * d[i - 1] + sinr * e[i - 2]
                    e[i - 2] = cosr * e[i - 2] - sinr * d[i - 1]
                    g = sinr * d[i - 2]
                    d[i - 2] = cosr * d[i - 2]
                    cosl, sinl, r = dlartg(f, g, old)
                    d[i - 1] = r
                    f = cosl * e[i - 2] + sinl * d[i - 2]
                    d[i - 2] = cosl * d[i - 2] - sinl * e[i - 2]
                    if i > ll + 1:
                        g = sinl * e[i - 3]
                        e[i - 3] = cosl * e[i - 3]
                    j = i - ll - 1
                    c1[j], s1[j], c2[j], s2[j] = cosr, -sinr, cosl, -sinl
                e[ll - 1] = f
                if abs(e[ll - 1]) <= thresh:
                    e[ll - 1] = 0.0
                dlasr_lvb(VT, rows, c2, s2)
    for i in range(n):
        if d[i] < 0.0:
            d[i] = -d[i]
            VT[i, :] = -VT[i, :]
    for i in range(n - 1):
        isub = 0
        smin = d[0]
        for j in range(1, n - i):
            if d[j] <= smin:
                isub, smin = j, d[j]
        if isub != n - 1 - i:
            d[isub], d[n - 1 - i] = d[n - 1 - i], smin
            VT[[isub, n - 1 - i]] = VT[[n - 1 - i, isub]]
    return d, VT


def _lastv(v):
    k = len(v)
    while k > 0 and v[k - 1] == 0.0:
        k -= 1
    return k


def _iladlc(m, n, C):
    if n == 0 or C[0, n - 1] != 0.0 or C[m - 1, n - 1] != 0.0:
        return n
    for j in range(n - 1, -1, -1):
        if any(C[i, j] != 0.0 for i in range(m)):
            return j + 1
    return 0


def _iladlr(m, n, C):
    if m == 0 or C[m - 1, 0] != 0.0 or C[m - 1, n - 1] != 0.0:
        return m
    r = 0
    for j in range(n):
        i = m
        while i >= 1 and C[i - 1, j] == 0.0:
            i -= 1
        r = max(r, i)
    return r


def _dlasdq_dbdsdc_sorts(d, VT):
    """dlasdq's selection sort (smallest first, strict <), then dbdsdc's
    (largest first, strict >).  Both are no-ops unless singular values tie
    exactly; the probe against LAPACK's dbdsdc pins the tie order."""
    n = len(d)
    d = list(d)
    for i in range(n):
        isub, smin = i, d[i]
        for j in range(i + 1, n):
            if d[j] < smin:
                isub, smin = j, d[j]
        if isub != i:
            d[isub], d[i] = d[i], smin
            VT[[isub, i]] = VT[[i, isub]]
    for i in range(n - 1):
        kk, p = i, d[i]
        for j in range(i + 1, n):
            if d[j] > p:
                kk, p = j, d[j]
        if kk != i:
            d[kk], d[i] = d[i], p
            VT[[kk, i]] = VT[[i, kk]]
    return d, VT


def dlarf_left(v, tau, C):
    if tau == 0.0:
        return
    lv = _lastv(v)
    if lv == 0:
        return
    lc = _iladlc(lv, C.shape[1], C)
    if lc == 0:
        return
    w = gemv_t(C[:lv, :lc], v[:lv])
    sub = C[:lv, :lc]
    ger(sub, v[:lv], w, -tau)


def dlarf_right(v, tau, C):
    if tau == 0.0:
        return
    lv = _lastv(v)
    if lv == 0:
        return
    lc = _iladlr(C.shape[0], lv, C)
    if lc == 0:
        return
    w = gemv_n(C[:lc, :lv], v[:lv])
    sub = C[:lc, :lv]
    ger(sub, w, v[:lv], -tau)


def svd_vt(A, old=False):
    """V^T of the m x 3 matrix A the way LAPACK dgesdd (JOBZ='S') gets it."""
    A = np.array(A, dtype=np.float64)
    m, n = A.shape
    if m >= 5:  # MNTHR = int(3 * 11 / 6): QR first, then bidiagonalise R
        for i in range(n):
            beta, tau, x = dlarfg(A[i, i], list(A[i + 1:, i]))
            A[i + 1:, i] = x
            A[i, i] = beta
            if i < n - 1 and tau != 0.0:
                aii = A[i, i]
                A[i, i] = 1.0
                dlarf_left(A[i:, i].copy(), tau, A[i:, i + 1:])
                A[i, i] = aii
        R = np.triu(A[:n, :n])
    else:
        R = A
    m2 = R.shape[0]
    d = [0.0] * n
    e = [0.0] * (n - 1)
    taup = [0.0] * n
    for i in range(n):
        beta, tq, x = dlarfg(R[i, i], list(R[i + 1:, i]))
        R[i + 1:, i] = x
        d[i] = beta
        R[i, i] = 1.0
        if i < n - 1:
            dlarf_left(R[i:, i].copy(), tq, R[i:, i + 1:])
        R[i, i] = d[i]
        if i < n - 1:
            beta, tp, x = dlarfg(R[i, i + 1], list(R[i, i + 2:]))
            R[i, i + 2:] = x
            e[i] = beta
            taup[i] = tp
            R[i, i + 1] = 1.0
            dlarf_right(R[i, i + 1:].copy(), tp, R[i + 1:, i + 1:])
            R[i, i + 1] = e[i]
    VT = np.eye(n)
    d, VT = dbdsqr(d, e, VT, old)
    d, VT = _dlasdq_dbdsdc_sorts(d, VT)
    # dormbr('P','R','T'): VT(:,2:3) := VT(:,2:3) * H(1) (H(2) has tau 0)
    v = np.array([1.0, R[0, 2]])
    dlarf_right(v, taup[0], VT[:, 1:])
    return np.array(d), VT
