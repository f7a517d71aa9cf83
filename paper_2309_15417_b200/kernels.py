"""Drop-in for the row kernels of `ltsdem.kernels` (kernels.py:23-201) and the
row helpers of `ltsdem.ccd`, evaluated by libltsgpu.so on the GPU.

Inputs are numpy arrays (or anything `np.asarray` accepts) with the
reference's shapes; outputs are numpy arrays, bit-identical to the
reference.  Each call copies its rows to the device, launches one kernel
and copies the result back.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _dev(x, shape_tail):
    torch = _lib.require_cuda()
    a = np.require(np.atleast_2d(np.asarray(x, dtype=np.float64)), requirements=["C", "W"])
    a = a.reshape(-1, *shape_tail)
    return torch.from_numpy(a).to(torch.device("cuda", torch.cuda.current_device())), len(a)


def _out(n, *tail, dtype=None):
    import torch
    return torch.empty((n, *tail), dtype=dtype or torch.float64,
                       device=torch.device("cuda", torch.cuda.current_device()))


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return C.c_void_p(t.data_ptr() if t.numel() else 0)


def _broadcast_rows(*xs):
    arrs = [np.atleast_2d(np.asarray(x, dtype=np.float64)) for x in xs]
    n = max(len(a) for a in arrs)
    return [np.broadcast_to(a, (n, 3)) for a in arrs]


def point_triangle_closest(p, a, b, c):
    """(dist (n,), closest (n,3)) of p to triangle abc per row (kernels.py:23-75)."""
    p, a, b, c = _broadcast_rows(p, a, b, c)
    (tp, n), (ta, _), (tb, _), (tc, _) = (_dev(x, (3,)) for x in (p, a, b, c))
    d, q = _out(n), _out(n, 3)
    _lib.check(_lib.lib().ltsg_point_triangle_closest(_p(tp), _p(ta), _p(tb), _p(tc), n, _p(d), _p(q),
                                                      _stream()), "point_triangle_closest")
    return d.cpu().numpy(), q.cpu().numpy()


def segment_segment_closest(p1, q1, p2, q2):
    """(dist, c1, c2) closest points of two segments per row (kernels.py:78-115)."""
    p1, q1, p2, q2 = _broadcast_rows(p1, q1, p2, q2)
    (a, n), (b, _), (c, _), (e, _) = (_dev(x, (3,)) for x in (p1, q1, p2, q2))
    d, c1, c2 = _out(n), _out(n, 3), _out(n, 3)
    _lib.check(_lib.lib().ltsg_segment_segment_closest(_p(a), _p(b), _p(c), _p(e), n, _p(d), _p(c1),
                                                       _p(c2), _stream()), "segment_segment_closest")
    return d.cpu().numpy(), c1.cpu().numpy(), c2.cpu().numpy()


def feature_distances(tri_a, tri_b):
    """ccd._feature_distances: row-wise 15-feature distance of (n,3,3) pairs."""
    (ta, n), (tb, m) = _dev(tri_a, (3, 3)), _dev(tri_b, (3, 3))
    if n != m:
        raise ValueError(f"row count mismatch: {n} vs {m}")
    d = _out(n)
    _lib.check(_lib.lib().ltsg_feature_distances(_p(ta), _p(tb), n, _p(d), _stream()),
               "feature_distances")
    return d.cpu().numpy()


def closest_feature(tri_a, tri_b):
    """ccd._closest_feature per row: (dist, pa, pb)."""
    (ta, n), (tb, _) = _dev(tri_a, (3, 3)), _dev(tri_b, (3, 3))
    d, pa, pb = _out(n), _out(n, 3), _out(n, 3)
    _lib.check(_lib.lib().ltsg_closest_feature(_p(ta), _p(tb), n, _p(d), _p(pa), _p(pb), _stream()),
               "closest_feature")
    return d.cpu().numpy(), pa.cpu().numpy(), pb.cpu().numpy()


def overlap_centroids(tri_a, tri_b, normal):
    """Row-batched triangle_overlap_centroid: (centroids (n,3), has (n,) bool)."""
    import torch

    (ta, n), (tb, _), (nm, _) = _dev(tri_a, (3, 3)), _dev(tri_b, (3, 3)), _dev(normal, (3,))
    c, h = _out(n, 3), _out(n, dtype=torch.int32)
    _lib.check(_lib.lib().ltsg_overlap_centroid(_p(ta), _p(tb), _p(nm), n, _p(c), _p(h), _stream()),
               "overlap_centroid")
    return c.cpu().numpy(), h.cpu().numpy() != 0


def triangle_overlap_centroid(tri_a, tri_b, normal):
    """kernels.triangle_overlap_centroid (kernels.py:138-201): centroid or None."""
    c, h = overlap_centroids(np.asarray(tri_a)[None], np.asarray(tri_b)[None], np.asarray(normal)[None])
    return c[0] if h[0] else None
