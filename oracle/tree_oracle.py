"""CPU oracle of surrogate-tree construction.  TEST INFRASTRUCTURE: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import it;
the product builds trees on the GPU (`paper_2309_15417_b200/treebuild.py`,
csrc/tree.cu) and has no CPU path.

Restates `ltsdem.surrogate.build_surrogate_tree` (surrogate.py:71-119) with
`_fit_parent_triangle` (surrogate.py:49-68) and `kernels.morton_order`
(kernels.py:118-135), vectorised over the groups of a level.  The
arithmetic matches the reference op for op (centroids by sequential row
sums, the 3x3 `dgemv` order ``fma(r2,u2, fma(r0,u0, r1*u1))`` for
``rel @ u``, batched LAPACK SVD which equals the per-group call).

Pinned: `tests/test_tree_oracle.py` checks it bit for bit against trees the
reference itself built (tests/golden/trees_gpu.npz, trees.npz; generator
tests/golden/make_golden_trees.py).  The plane fit calls numpy's SVD, i.e.
the host's LAPACK; `oracle/lapack_svd.py` restates that routine explicitly
and is what csrc/lapack3.cuh implements.
"""

from __future__ import annotations

import numpy as np

from paper_2309_15417_b200.bodies import ChildIndex, SurrogateLevel, SurrogateTree

_EPS_PAD = 1e-12
_TINY = 1e-300


def morton_order(points: np.ndarray, bits: int = 10) -> np.ndarray:
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    lo = pts.min(axis=0)
    span = pts.max(axis=0) - lo
    span[span <= 0.0] = 1.0
    q = ((pts - lo) * ((2 ** bits - 1) / span)).astype(np.uint64)
    code = np.zeros(len(pts), dtype=np.uint64)
    for i in range(bits):
        for axis in range(3):
            code |= ((q[:, axis] >> np.uint64(i)) & np.uint64(1)) << np.uint64(3 * i + axis)
    return np.argsort(code, kind="stable")


def _fma(a, b, c):
    # exact FMA for the 3-term dgemv order; see oracle-independent note above
    from ._fma import fma
    return fma(a, b, c)


def _dgemv_rows(rel: np.ndarray, u: np.ndarray) -> np.ndarray:
    """(G, m, 3) @ (G, 3) per group, in OpenBLAS dgemv order."""
    u = u[:, None, :]
    return _fma(rel[..., 2], u[..., 2], _fma(rel[..., 0], u[..., 0], rel[..., 1] * u[..., 1]))


def _row_mean(pts: np.ndarray, axis: int) -> np.ndarray:
    """numpy mean over a short strided axis: sequential sum, then divide."""
    n = pts.shape[axis]
    acc = np.take(pts, 0, axis=axis).copy()
    for i in range(1, n):
        acc = acc + np.take(pts, i, axis=axis)
    return acc / n


def _fit_parents(points: np.ndarray) -> np.ndarray:
    """Parent triangle per group of points (G, m, 3) -> (G, 3, 3)."""
    centroid = _row_mean(points, 1)
    rel = points - centroid[:, None, :]
    _, _, vt = np.linalg.svd(rel, full_matrices=False)
    u, v = vt[:, 0], vt[:, 1]
    su = _dgemv_rows(rel, u)
    sv = _dgemv_rows(rel, v)
    spread = np.abs(rel).max(axis=(1, 2))
    spread = np.where(spread == 0.0, 1.0, spread)
    pad = np.maximum(1e-9, 1e-6 * spread)
    lo_u = su.min(axis=1) - pad
    hi_u = su.max(axis=1) + pad
    lo_v = sv.min(axis=1) - pad
    hi_v = sv.max(axis=1) + pad
    w = hi_u - lo_u
    h = hi_v - lo_v
    p0 = (centroid + lo_u[:, None] * u) + lo_v[:, None] * v
    return np.stack([p0, p0 + (2.0 * w)[:, None] * u, p0 + (2.0 * h)[:, None] * v], axis=1)


def _point_triangle_dist(p, a, b, c):
    """kernels.point_triangle_closest distance only (kernels.py:23-75)."""
    def dot(x, y):
        return (x[..., 0] * y[..., 0] + x[..., 2] * y[..., 2]) + x[..., 1] * y[..., 1]

    def sdiv(n, d):
        return n / np.where(np.abs(d) > _TINY, d, 1.0)

    ab, ac, ap, bp, cp = b - a, c - a, p - a, p - b, p - c
    d1, d2, d3, d4, d5, d6 = dot(ab, ap), dot(ac, ap), dot(ab, bp), dot(ac, bp), dot(ab, cp), dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    denom = (va + vb) + vc
    out = (a + ab * sdiv(vb, denom)[..., None]) + ac * sdiv(vc, denom)[..., None]
    m = (va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0)
    out = np.where(m[..., None], b + sdiv(d4 - d3, (d4 - d3) + (d5 - d6))[..., None] * (c - b), out)
    m = (vb <= 0) & (d2 >= 0) & (d6 <= 0)
    out = np.where(m[..., None], a + sdiv(d2, d2 - d6)[..., None] * ac, out)
    m = (vc <= 0) & (d1 >= 0) & (d3 <= 0)
    out = np.where(m[..., None], a + sdiv(d1, d1 - d3)[..., None] * ab, out)
    out = np.where(((d6 >= 0) & (d5 <= d6))[..., None], c, out)
    out = np.where(((d3 >= 0) & (d4 <= d3))[..., None], b, out)
    out = np.where(((d1 <= 0) & (d2 <= 0))[..., None], a, out)
    w = p - out
    return np.sqrt((w[..., 0] * w[..., 0] + w[..., 1] * w[..., 1]) + w[..., 2] * w[..., 2])


def build_surrogate_tree(corners, epsilon: float, fanout: int = 4,
                         max_levels: int = 8) -> SurrogateTree:
    """Morton-grouped coarsening hierarchy (surrogate.py:71-119)."""
    if epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    if fanout < 2:
        raise ValueError(f"fanout must be at least 2, got {fanout}")
    corners = np.ascontiguousarray(np.asarray(corners, dtype=np.float64).reshape(-1, 3, 3))
    levels = [SurrogateLevel(corners=corners, epsilon=np.full(len(corners), float(epsilon)),
                             children=None)]
    while levels[-1].size > 1 and len(levels) < max_levels:
        fine = levels[-1]
        order = morton_order(_row_mean(fine.corners, 1))
        n_full = len(order) // fanout
        groups = [order[i:i + fanout] for i in range(0, len(order), fanout)]
        parents = np.empty((len(groups), 3, 3))
        peps = np.empty(len(groups))
        spans = []
        if n_full:
            spans.append((0, n_full, order[:n_full * fanout].reshape(n_full, fanout)))
        if len(order) % fanout:
            spans.append((n_full, n_full + 1, order[n_full * fanout:].reshape(1, -1)))
        for g0, g1, idx in spans:
            pts = fine.corners[idx].reshape(g1 - g0, -1, 3)
            tri = _fit_parents(pts)
            m = pts.shape[1]
            dist = _point_triangle_dist(
                pts,
                np.broadcast_to(tri[:, None, 0], (g1 - g0, m, 3)),
                np.broadcast_to(tri[:, None, 1], (g1 - g0, m, 3)),
                np.broadcast_to(tri[:, None, 2], (g1 - g0, m, 3)))
            child_eps = np.repeat(fine.epsilon[idx], 3, axis=1)
            parents[g0:g1] = tri
            peps[g0:g1] = (dist + child_eps).max(axis=1) + _EPS_PAD
        children = [np.sort(g) for g in groups]
        levels.append(SurrogateLevel(corners=parents, epsilon=peps, children=children))
    return SurrogateTree(levels=levels)


def _morton_codes(points: np.ndarray, bits: int = 10) -> np.ndarray:
    """Row-batched Morton codes of (P, n, 3) points, as morton_order computes them."""
    lo = points.min(axis=1, keepdims=True)
    span = points.max(axis=1, keepdims=True) - lo
    span[span <= 0.0] = 1.0
    q = ((points - lo) * ((2 ** bits - 1) / span)).astype(np.uint64)
    code = np.zeros(points.shape[:2], dtype=np.uint64)
    for i in range(bits):
        for axis in range(3):
            code |= ((q[..., axis] >> np.uint64(i)) & np.uint64(1)) << np.uint64(3 * i + axis)
    return code


def build_surrogate_trees(corners, epsilon: float, fanout: int = 4, max_levels: int = 8) -> list:
    """build_surrogate_tree for P meshes with the same triangle count at once.

    `corners` is (P, n, 3, 3).  Every operation is the per-tree one applied
    along a leading batch axis (Morton codes, stable argsort, batched LAPACK
    SVD, the dgemv-ordered projections), so each tree equals the one
    build_surrogate_tree gives for that mesh alone.  Children are stored as
    a compact CSR index (ChildIndex) instead of one array per parent.
    """
    corners = np.ascontiguousarray(np.asarray(corners, dtype=np.float64))
    P, n = corners.shape[:2]
    if epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    levels = [[SurrogateLevel(corners=corners[p], epsilon=np.full(n, float(epsilon)), children=None)]
              for p in range(P)]
    cur = corners
    cur_eps = np.full((P, n), float(epsilon))
    size = n
    depth = 1
    while size > 1 and depth < max_levels:
        order = np.argsort(_morton_codes(_row_mean(cur, 2)), axis=1, kind="stable")
        n_full = size // fanout
        rem = size % fanout
        G = n_full + (1 if rem else 0)
        parents = np.empty((P, G, 3, 3))
        peps = np.empty((P, G))
        parts = []
        if n_full:
            parts.append((0, n_full, order[:, :n_full * fanout].reshape(P, n_full, fanout)))
        if rem:
            parts.append((n_full, G, order[:, n_full * fanout:].reshape(P, 1, rem)))
        for g0, g1, idx in parts:
            gsz = idx.shape[2]
            rows = np.take_along_axis(cur, idx.reshape(P, -1)[..., None, None], axis=1)
            pts = rows.reshape(P * (g1 - g0), gsz * 3, 3)
            tri = _fit_parents(pts)
            m = pts.shape[1]
            dist = _point_triangle_dist(
                pts,
                np.broadcast_to(tri[:, None, 0], (len(pts), m, 3)),
                np.broadcast_to(tri[:, None, 1], (len(pts), m, 3)),
                np.broadcast_to(tri[:, None, 2], (len(pts), m, 3)))
            ceps = np.take_along_axis(cur_eps, idx.reshape(P, -1), axis=1).reshape(len(pts), gsz)
            child_eps = np.repeat(ceps, 3, axis=1)
            parents[:, g0:g1] = tri.reshape(P, g1 - g0, 3, 3)
            peps[:, g0:g1] = ((dist + child_eps).max(axis=1) + _EPS_PAD).reshape(P, g1 - g0)
        srt = np.sort(order, axis=1)
        if rem:
            kids_full = np.sort(order[:, :n_full * fanout].reshape(P, n_full, fanout), axis=2)
            kids_rem = np.sort(order[:, n_full * fanout:], axis=1)
        else:
            kids_full = np.sort(order.reshape(P, n_full, fanout), axis=2)
        ptr = np.concatenate([np.arange(0, n_full * fanout + 1, fanout), [size]] if rem else
                             [np.arange(0, n_full * fanout + 1, fanout)]).astype(np.int64)
        del srt
        for p in range(P):
            flat = kids_full[p].reshape(-1)
            if rem:
                flat = np.concatenate([flat, kids_rem[p]])
            levels[p].append(SurrogateLevel(corners=parents[p], epsilon=peps[p],
                                            children=ChildIndex(ptr, flat.astype(np.int64))))
        cur = parents
        cur_eps = peps
        size = G
        depth += 1
    return [SurrogateTree(levels=lv) for lv in levels]


def build_many(corners_list, epsilons, fanout: int = 4, max_levels: int = 8) -> list:
    """Trees of arbitrary meshes (the signature of treebuild.build_surrogate_trees):
    meshes with equal triangle count and epsilon go through the batched builder."""
    corners_list = [np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1, 3, 3)) for c in corners_list]
    eps = np.broadcast_to(np.asarray(epsilons, dtype=np.float64), (len(corners_list),))
    groups = {}
    for k, c in enumerate(corners_list):
        groups.setdefault((len(c), float(eps[k])), []).append(k)
    out = [None] * len(corners_list)
    for (n, e), idx in groups.items():
        for lo in range(0, len(idx), 256):
            part = idx[lo:lo + 256]
            trees = build_surrogate_trees(np.stack([corners_list[k] for k in part]), e, fanout=fanout,
                                          max_levels=max_levels)
            for k, t in zip(part, trees):
                out[k] = t
    return out
