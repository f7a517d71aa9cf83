"""Correctly rounded fused multiply-add for float64 numpy arrays.

Used only by the tree oracle (`tree_oracle.py`) to reproduce
OpenBLAS's FMA-based `dgemv` order.  Error-free product (Dekker/Veltkamp)
and sum (Knuth TwoSum); the two low parts are combined with
round-to-odd before the final rounding, which makes the result correctly
rounded (Boldo & Melquiond 2008).
"""

from __future__ import annotations

import numpy as np

_C = 134217729.0  # 2**27 + 1


def fma(a, b, c):
    a, b, c = np.broadcast_arrays(*(np.asarray(x, dtype=np.float64) for x in (a, b, c)))
    p = a * b
    t = _C * a
    ah = t - (t - a)
    al = a - ah
    t = _C * b
    bh = t - (t - b)
    bl = b - bh
    pe = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    s = c + p
    z = s - c
    se = (c - (s - z)) + (p - z)
    lo = se + pe
    z = lo - se
    le = (se - (lo - z)) + (pe - z)
    odd = (le != 0.0) & ((lo.view(np.int64) & 1) == 0)
    lo = np.where(odd, np.nextafter(lo, np.where(le > 0.0, np.inf, -np.inf)), lo)
    out = s + lo
    plain = ~np.isfinite(p) | (p == 0.0)
    return np.where(plain, p + c, out)
