"""TEST INFRASTRUCTURE ONLY -- never imported by the product package.

Exact-rounding helpers for the CPU oracle (`oracle/narrow_oracle.py`).

The reference (`ltsdem`, pure numpy) reaches three kinds of arithmetic whose
rounding order is decided by library code rather than by its own source:

* `np.einsum` row dots (`kernels.py:15-16`, `ccd.py:132`): on C-contiguous
  rows numpy's SIMD inner loop sums a length-3 dot as ``(x0*y0 + x2*y2) +
  x1*y1``; on non-C-contiguous rows (`_closest_feature`, `ccd.py:158-162`)
  it is the sequential ``(x0*y0 + x1*y1) + x2*y2``.  Never contracted to FMA.
* OpenBLAS (`@` on 1-D / 2-D operands, 1-D `np.linalg.norm`): `ddot` and the
  3x3 `dgemm` are the FMA chain ``fma(x2,y2, fma(x1,y1, x0*y0))``; the 3x3
  `dgemv` (``M @ v``) is ``fma(m2,v2, fma(m0,v0, m1*v1))``.
* numpy reductions: `axis` reductions over a strided axis are sequential,
  1-D `sum` is numpy's 8-way pairwise sum.

These orders were probed in the build container (numpy 2.3.5, OpenBLAS
0.3.30 SkylakeX kernels) and are pinned by the golden vectors in
`tests/golden/`, which were produced by the reference itself.  Writing them
out explicitly here makes the oracle independent of the host it runs on
(the GPU box may select other OpenBLAS kernels).

`fma` is emulated exactly in numpy (Boldo & Melquiond, "Emulation of FMA and
correctly rounded sums: proved algorithms using rounding to odd", IEEE TC
2008): exact product by Veltkamp/Dekker splitting, exact sum by TwoSum, the
low parts combined with round-to-odd, one final round-to-nearest.
"""

from __future__ import annotations

import numpy as np

_SPLITTER = 134217729.0  # 2**27 + 1


def _two_prod(a, b):
    p = a * b
    t = _SPLITTER * a
    ah = t - (t - a)
    al = a - ah
    t = _SPLITTER * b
    bh = t - (t - b)
    bl = b - bh
    err = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, err


def _two_sum(a, b):
    s = a + b
    bv = s - a
    err = (a - (s - bv)) + (b - bv)
    return s, err


def _add_round_odd(a, b):
    s, err = _two_sum(a, b)
    inexact_even = (err != 0.0) & ((s.view(np.int64) & 1) == 0)
    toward = np.where(err > 0.0, np.inf, -np.inf)
    return np.where(inexact_even, np.nextafter(s, toward), s)


def fma(a, b, c):
    """Correctly rounded a*b + c, elementwise, in plain float64 numpy."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    a, b, c = np.broadcast_arrays(a, b, c)
    ph, pl = _two_prod(a, b)
    sh, sl = _two_sum(c, ph)
    # a*b with zero / inf operands: the splitting is not needed and may
    # produce nan; fall back to the plain product-sum which is then exact.
    out = sh + _add_round_odd(sl, pl)
    plain = ~np.isfinite(ph) | (ph == 0.0)
    if plain.any():
        out = np.where(plain, ph + c, out)
    return out


def dot_simd(u, v):
    """einsum row dot on C-contiguous rows: (x0*y0 + x2*y2) + x1*y1."""
    return (u[..., 0] * v[..., 0] + u[..., 2] * v[..., 2]) + u[..., 1] * v[..., 1]


def dot_seq(u, v):
    """einsum row dot on non-contiguous rows: (x0*y0 + x1*y1) + x2*y2."""
    return (u[..., 0] * v[..., 0] + u[..., 1] * v[..., 1]) + u[..., 2] * v[..., 2]


def dot_blas(u, v):
    """OpenBLAS ddot for n=3: fma(x2,y2, fma(x1,y1, x0*y0))."""
    return fma(u[..., 2], v[..., 2], fma(u[..., 1], v[..., 1], u[..., 0] * v[..., 0]))


def norm_rows(w):
    """np.linalg.norm(w, axis=-1): sqrt((x0^2 + x1^2) + x2^2)."""
    return np.sqrt((w[..., 0] * w[..., 0] + w[..., 1] * w[..., 1]) + w[..., 2] * w[..., 2])


def norm_blas(w):
    """1-D np.linalg.norm = sqrt(ddot(w, w))."""
    return np.sqrt(dot_blas(w, w))


def matmul3_blas(m, b):
    """(..., 3, 3) @ (3, 3) through OpenBLAS dgemm: per entry an FMA chain over k."""
    m = np.asarray(m, dtype=np.float64)
    out = np.empty(np.broadcast_shapes(m.shape, (3, 3)))
    for i in range(3):
        for j in range(3):
            out[..., i, j] = fma(m[..., i, 2], b[2, j],
                                 fma(m[..., i, 1], b[1, j], m[..., i, 0] * b[0, j]))
    return out


def matvec3_blas(m, v):
    """(3, 3) @ (3,) through OpenBLAS dgemv: fma(m2,v2, fma(m0,v0, m1*v1))."""
    return np.array([
        float(fma(m[i, 2], v[2], fma(m[i, 0], v[0], m[i, 1] * v[1]))) for i in range(3)
    ])


def cross3(a, b):
    """np.cross on 3-vectors: a1*b2 - a2*b1, ... (no FMA)."""
    return np.stack([
        a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
        a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
        a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0],
    ], axis=-1)


def pairwise_sum(values) -> float:
    """numpy's 1-D float64 `sum` (pairwise_sum with 8 partial accumulators)."""
    a = [float(x) for x in values]
    n = len(a)
    if n < 8:
        acc = 0.0
        for x in a:
            acc += x
        return acc
    if n > 128:
        raise NotImplementedError("only short polygon sums are needed")
    r = a[:8]
    i = 8
    while i < n - (n % 8):
        for j in range(8):
            r[j] += a[i + j]
        i += 8
    acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        acc += a[i]
        i += 1
    return acc


def round9(x) -> float:
    """`round(np.float64(x), 9)` as the reference's sort key evaluates it
    (ccd.py:541-542): numpy rounds by ``rint(x * 1e9) / 1e9`` -- not
    Python's correctly rounded decimal rounding."""
    return float(np.rint(np.float64(x) * 1e9) / 1e9)
