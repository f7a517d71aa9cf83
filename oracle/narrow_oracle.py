"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the narrow phase.

A numpy restatement of the reference narrow phase (`ltsdem`, pure
Python/numpy), used by `tests/` as the checker, by `__graft_entry__.smoke()`
as the checker, and by `bench.py --impl reference` / the `cpu_baseline`
leg as the CPU baseline.  The product package (`paper_2309_15417_b200`)
never imports this module.

What it restates (file:line under /root/reference/pkg/src/ltsdem):

* row-batched closest points: `kernels.point_triangle_closest`
  (kernels.py:23-75), `kernels.segment_segment_closest` (kernels.py:78-115)
* the 15-feature triangle-pair distance `ccd._feature_distances`
  (ccd.py:135-153) and its witness variant `ccd._closest_feature`
  (ccd.py:156-174)
* free-flight rigid motion `ccd._Motion` (ccd.py:82-132) with
  `quaternions.to_matrix` (quaternions.py:54-63)
* the multiscale search `ccd._search` (ccd.py:373-487) including the
  sampling screen `_evaluate` (ccd.py:321-370), certified zoom
  `_isolate_crossings` (ccd.py:242-308) and bisection `_batched_bisect`
  (ccd.py:311-318)
* contact records `_make_contact` / `_face_normal` (ccd.py:177-213) with
  `kernels.triangle_overlap_centroid` (kernels.py:138-201)
* contact fusion `ccd.filter_contacts` (ccd.py:527-577)
* public entries `pair_earliest_contact` (ccd.py:490-502) and
  `compute_effective_dt` (ccd.py:505-524)

The search is organised differently from the reference (a vectorised
frontier per level pair instead of per-candidate Python lists), but every
floating-point operation is the one the reference performs, in the same
order (see `fpexact.py` for the library-decided orders).  Parity of this
restatement with the reference is pinned by `tests/golden/*` (produced by
the reference itself, script `tests/golden/make_golden.py`) and checked by
`tests/test_oracle_golden.py`.

Inputs are duck-typed like the reference's: a body has `pid` (dynamic,
with `timeline.current`) or `sid` (static), and `tree.levels[l]` with
`corners (k,3,3)`, `epsilon (k,)`, `children` (list of int arrays).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fpexact import (
    cross3, dot_blas, dot_seq, dot_simd, fma, matmul3_blas, matvec3_blas, norm_blas,
    norm_rows, pairwise_sum, round9,
)

# ccd.py:29-36, kernels.py:12
WIDEN = 1e-3
REST_SLOP = 1e-9
MIN_SAMPLES = 2
MAX_SAMPLES = 33
ZOOM_SAMPLES = 17
GRAZE_TOL = 1e-9
BISECT_ITERS = 52
PARALLEL_COS = 1.0 - 1e-3
TINY = 1e-300

# feature tables (ccd.py:38-40): edge i of a triangle runs corner i -> corner i+1
_EA = np.repeat(np.arange(3), 3)
_EB = np.tile(np.arange(3), 3)
_NXT = np.array([1, 2, 0])


# --------------------------------------------------------------------------
# primitive closest-point queries (kernels.py)
# --------------------------------------------------------------------------

def _sdiv(num, den):
    return num / np.where(np.abs(den) > TINY, den, 1.0)


def _clip01(x):
    return np.clip(x, 0.0, 1.0)


# region codes in increasing priority; kernels.py:49-72 overwrites in this order
FACE, EDGE_BC, EDGE_AC, EDGE_AB, VERT_C, VERT_B, VERT_A = range(7)


def point_triangle(p, a, b, c, dot=dot_simd):
    """Closest point on triangle abc to p, rows independent (kernels.py:23-75).

    Returns (distance, closest, region) -- the region code is extra output
    used by the tests and by the flop accounting.
    """
    p, a, b, c = (np.atleast_2d(np.asarray(x, dtype=np.float64)) for x in (p, a, b, c))
    ab = b - a
    ac = c - a
    ap = p - a
    bp = p - b
    cp = p - c
    d1, d2 = dot(ab, ap), dot(ac, ap)
    d3, d4 = dot(ab, bp), dot(ac, bp)
    d5, d6 = dot(ab, cp), dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4

    region = np.full(len(p), FACE)
    bc_num, bc_rest = d4 - d3, d5 - d6
    region[(va <= 0) & (bc_num >= 0) & (bc_rest >= 0)] = EDGE_BC
    region[(vb <= 0) & (d2 >= 0) & (d6 <= 0)] = EDGE_AC
    region[(vc <= 0) & (d1 >= 0) & (d3 <= 0)] = EDGE_AB
    region[(d6 >= 0) & (d5 <= d6)] = VERT_C
    region[(d3 >= 0) & (d4 <= d3)] = VERT_B
    region[(d1 <= 0) & (d2 <= 0)] = VERT_A

    denom = (va + vb) + vc
    out = (a + ab * _sdiv(vb, denom)[:, None]) + ac * _sdiv(vc, denom)[:, None]
    sel = region == EDGE_BC
    out[sel] = b[sel] + _sdiv(bc_num, bc_num + bc_rest)[sel, None] * (c[sel] - b[sel])
    sel = region == EDGE_AC
    out[sel] = a[sel] + _sdiv(d2, d2 - d6)[sel, None] * ac[sel]
    sel = region == EDGE_AB
    out[sel] = a[sel] + _sdiv(d1, d1 - d3)[sel, None] * ab[sel]
    for code, corner in ((VERT_C, c), (VERT_B, b), (VERT_A, a)):
        sel = region == code
        out[sel] = corner[sel]
    return norm_rows(p - out), out, region


def segment_segment(p1, q1, p2, q2):
    """Clamped closest points of segments [p1,q1], [p2,q2] (kernels.py:78-115)."""
    p1, q1, p2, q2 = (np.atleast_2d(np.asarray(x, dtype=np.float64)) for x in (p1, q1, p2, q2))
    u = q1 - p1
    w = q2 - p2
    r = p1 - p2
    uu = dot_simd(u, u)
    ww = dot_simd(w, w)
    wr = dot_simd(w, r)
    ur = dot_simd(u, r)
    uw = dot_simd(u, w)
    det = uu * ww - uw * uw

    s = _clip01(_sdiv(uw * wr - ur * ww, det))
    s = np.where(det > 1e-14 * uu * ww + TINY, s, 0.0)  # parallel rows take s = 0
    t = _sdiv(uw * s + wr, ww)
    s_lo = _clip01(_sdiv(-ur, uu))
    s_hi = _clip01(_sdiv(uw - ur, uu))
    s = np.where(t < 0.0, s_lo, s)
    s = np.where(t > 1.0, s_hi, s)
    t = _clip01(t)
    u_dead = uu <= TINY
    w_dead = ww <= TINY
    s = np.where(u_dead, 0.0, s)
    t = np.where(u_dead, _clip01(_sdiv(wr, ww)), t)
    t = np.where(w_dead, 0.0, t)
    s = np.where(w_dead & ~u_dead, s_lo, s)
    c1 = p1 + s[:, None] * u
    c2 = p2 + t[:, None] * w
    return norm_rows(c1 - c2), c1, c2


# --------------------------------------------------------------------------
# triangle-pair distance (ccd.py:135-174)
# --------------------------------------------------------------------------

def tri_pair_distance(ta, tb):
    """Row-wise minimum over the 6 vertex-triangle and 9 edge-edge features."""
    ta = np.asarray(ta, dtype=np.float64)
    tb = np.asarray(tb, dtype=np.float64)
    best = None
    for pts, tri in ((ta, tb), (tb, ta)):
        for k in range(3):
            d, _, _ = point_triangle(pts[:, k], tri[:, 0], tri[:, 1], tri[:, 2])
            best = d if best is None else np.minimum(best, d)
    for ea, eb in zip(_EA, _EB):
        d, _, _ = segment_segment(ta[:, ea], ta[:, _NXT[ea]], tb[:, eb], tb[:, _NXT[eb]])
        best = np.minimum(best, d)
    return best


def tri_pair_witness(ta, tb):
    """Distance and witness points of the winning feature, one triangle pair.

    The reference builds its point-triangle operands from broadcast views
    (ccd.py:159-161), so those dots round sequentially (`dot_seq`); the
    segment operands are C-ordered fancy-index copies (`dot_simd`).
    Vertex-triangle wins ties (ccd.py:170).
    """
    ta = np.asarray(ta, dtype=np.float64)
    tb = np.asarray(tb, dtype=np.float64)
    pts = np.concatenate([ta, tb])
    tris = np.concatenate([np.broadcast_to(tb, (3, 3, 3)), np.broadcast_to(ta, (3, 3, 3))])
    d_vt, c_vt, _ = point_triangle(pts, tris[:, 0], tris[:, 1], tris[:, 2], dot=dot_seq)
    d_ee, e1, e2 = segment_segment(ta[_EA], ta[_NXT[_EA]], tb[_EB], tb[_NXT[_EB]])
    i = int(np.argmin(d_vt))
    j = int(np.argmin(d_ee))
    if d_vt[i] <= d_ee[j]:
        if i < 3:
            return float(d_vt[i]), pts[i].copy(), c_vt[i].copy()
        return float(d_vt[i]), c_vt[i].copy(), pts[i].copy()
    return float(d_ee[j]), e1[j].copy(), e2[j].copy()


def unit_face_normal(tri):
    n = cross3(tri[1] - tri[0], tri[2] - tri[0])
    ln = float(norm_blas(n))
    return n / ln if ln > 0.0 else np.array([0.0, 0.0, 1.0])


def _mean3(rows):
    return ((rows[0] + rows[1]) + rows[2]) / 3.0


def overlap_centroid(ta, tb, normal):
    """Sutherland-Hodgman overlap centroid of two near-parallel triangles
    lifted to their mid-plane, or None (kernels.py:138-201)."""
    n = normal / float(norm_blas(normal))
    helper = np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    u = cross3(n, helper)
    u = u / float(norm_blas(u))
    v = cross3(n, u)
    origin = _mean3(ta)

    def flat(tri):
        rel = tri - origin
        return [np.array([float(dot_blas(q, u)), float(dot_blas(q, v))]) for q in rel]

    poly = flat(tb)
    window = flat(ta)
    e1 = window[1] - window[0]
    e2 = window[2] - window[0]
    if e1[0] * e2[1] - e1[1] * e2[0] < 0.0:
        window = window[::-1]

    def inside(q, base, edge):
        return edge[0] * (q[1] - base[1]) - edge[1] * (q[0] - base[0]) >= -1e-12

    for i in range(3):
        if not poly:
            return None
        base = window[i]
        edge = window[(i + 1) % 3] - base
        clipped = []
        for j, cur in enumerate(poly):
            prev = poly[j - 1]
            cin = inside(cur, base, edge)
            if cin != inside(prev, base, edge):
                dv = cur - prev
                den = edge[0] * dv[1] - edge[1] * dv[0]
                if abs(den) > TINY:
                    lam = (edge[0] * (base[1] - prev[1]) - edge[1] * (base[0] - prev[0])) / -den
                    clipped.append(prev + np.clip(lam, 0.0, 1.0) * dv)
            if cin:
                clipped.append(cur)
        poly = clipped
    if len(poly) < 3:
        return None
    xy = np.array(poly)
    x, y = xy[:, 0], xy[:, 1]
    xn, yn = np.roll(x, -1), np.roll(y, -1)
    cr = x * yn - xn * y
    area = 0.5 * pairwise_sum(cr)
    if abs(area) < 1e-18:
        sx = xy[0].copy()
        for row in xy[1:]:
            sx = sx + row
        c2 = sx / len(xy)
    else:
        c2 = np.array([pairwise_sum((x + xn) * cr), pairwise_sum((y + yn) * cr)]) / (6.0 * area)
    lift_a = matvec3_blas(ta - origin, n)
    lift_b = matvec3_blas(tb - origin, n)
    mid = 0.5 * (((lift_a[0] + lift_a[1]) + lift_a[2]) / 3.0) \
        + 0.5 * (((lift_b[0] + lift_b[1]) + lift_b[2]) / 3.0)
    return ((origin + c2[0] * u) + c2[1] * v) + mid * n


# --------------------------------------------------------------------------
# rigid free flight (ccd.py:82-132)
# --------------------------------------------------------------------------

def quat_to_matrix(q):
    """quaternions.to_matrix (quaternions.py:54-63)."""
    w, x, y, z = (float(c) for c in q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


class RigidPath:
    """Constant-velocity, constant-spin motion of one body's surrogate tree."""

    def __init__(self, body):
        if hasattr(body, "timeline"):
            st = body.timeline.current
            self.bid = int(body.pid)
            self.x0 = np.asarray(st.position, dtype=np.float64).copy()
            self.v = np.asarray(st.velocity, dtype=np.float64).copy()
            spin = np.asarray(st.angular_velocity, dtype=np.float64)
            self.base = quat_to_matrix(st.rotation)
        else:
            self.bid = int(body.sid)
            self.x0 = np.zeros(3)
            self.v = np.zeros(3)
            spin = np.zeros(3)
            self.base = np.eye(3)
        self.tree = body.tree
        self.omega = float(norm_blas(spin))
        if self.omega > 0.0:
            k = spin / self.omega
            self.K = np.array([[0.0, -k[2], k[1]], [k[2], 0.0, -k[0]], [-k[1], k[0], 0.0]])
            self.KK = matmul3_blas(self.K, self.K)
        else:
            self.K = None
        self._arm = {}

    def arm(self, level):
        got = self._arm.get(level)
        if got is None:
            got = norm_rows(self.tree.levels[level].corners).max(axis=1)
            self._arm[level] = got
        return got

    def rotation_at(self, taus):
        taus = np.asarray(taus, dtype=np.float64)
        if self.K is None:
            return np.broadcast_to(self.base, (len(taus), 3, 3))
        ang = self.omega * taus
        s = np.sin(ang)[:, None, None]
        c = (1.0 - np.cos(ang))[:, None, None]
        m = (np.eye(3) + s * self.K) + c * self.KK
        return matmul3_blas(m, self.base)

    def world(self, level, tris, taus):
        """World corners (m,3,3): einsum('mij,mpj->mpi') + x0 + tau v."""
        taus = np.asarray(taus, dtype=np.float64)
        loc = self.tree.levels[level].corners[np.asarray(tris, dtype=np.int64)]
        rot = self.rotation_at(taus)
        pos = self.x0[None, :] + taus[:, None] * self.v[None, :]
        out = np.empty((len(taus), 3, 3))
        for i in range(3):
            out[:, :, i] = ((rot[:, None, i, 0] * loc[:, :, 0] + rot[:, None, i, 2] * loc[:, :, 2])
                            + rot[:, None, i, 1] * loc[:, :, 1]) + pos[:, None, i]
        return out


# --------------------------------------------------------------------------
# the search (ccd.py:321-487)
# --------------------------------------------------------------------------

def linspace_rows(start, stop, count):
    """Concatenated np.linspace(start[i], stop[i], count[i]) (count 1 -> [start]).

    numpy 2.x: step = (stop-start)/(n-1); g[i] = i*step + start; last = stop;
    a zero step falls back to g[i] = (i/(n-1))*delta + start.
    """
    start = np.asarray(start, dtype=np.float64)
    stop = np.broadcast_to(np.asarray(stop, dtype=np.float64), start.shape)
    count = np.asarray(count, dtype=np.int64)
    owner = np.repeat(np.arange(len(count)), count)
    first = np.cumsum(count) - count
    idx = np.arange(int(count.sum())) - first[owner]
    fi = idx.astype(np.float64)
    div = np.maximum(count - 1, 1).astype(np.float64)[owner]
    delta = (stop - start)[owner]
    step = delta / div
    g = np.where(step == 0.0, (fi / div) * delta, fi * step) + start[owner]
    last = (idx == count[owner] - 1) & (count[owner] > 1)
    g[last] = stop[owner][last]
    return g, owner, first


@dataclass
class Candidates:
    pair: np.ndarray
    ia: np.ndarray
    ib: np.ndarray
    w0: np.ndarray

    def __len__(self):
        return len(self.pair)


@dataclass
class SearchOutput:
    dt: float
    collision: bool
    first_contact: float | None
    narrowing_iters: int
    bound_history: list
    resting: list = field(default_factory=list)    # (pair, ia, ib, h)
    crossings: list = field(default_factory=list)  # (tau, pair, ia, ib, h)
    rows: int = 0            # screen rows evaluated (reference-equivalent tests)
    zoom_rows: int = 0
    bisect_rows: int = 0


def _pair_rows(paths, pairs, pair_idx, la, lb, ia, ib, taus):
    """World triangles of both sides for each row, grouped per body."""
    out = []
    for side, lvl, tri in ((0, la, ia), (1, lb, ib)):
        bids = np.array([pairs[k][side] for k in range(len(pairs))])[pair_idx]
        world = np.empty((len(taus), 3, 3))
        for bid in np.unique(bids):
            sel = bids == bid
            world[sel] = paths[int(bid)].world(lvl, tri[sel], taus[sel])
        out.append(world)
    return out


def _screen(paths, pairs, la, lb, cand: Candidates, dt: float):
    """Sample each candidate over [w0, dt] (ccd.py:321-370).  Never prunes by
    a narrowed bound: in the reference schedule the bound equals dt until
    the fine bucket, which is processed last (ccd.py:394)."""
    n = len(cand)
    h = np.empty(n)
    speed = np.empty(n)
    for k in np.unique(cand.pair):
        sel = cand.pair == k
        pa, pb = paths[pairs[k][0]], paths[pairs[k][1]]
        h[sel] = pa.tree.levels[la].epsilon[cand.ia[sel]] + pb.tree.levels[lb].epsilon[cand.ib[sel]]
        sp = np.full(int(sel.sum()), float(norm_blas(pa.v - pb.v)))
        if pa.omega > 0.0:
            sp = sp + pa.omega * pa.arm(la)[cand.ia[sel]]
        if pb.omega > 0.0:
            sp = sp + pb.omega * pb.arm(lb)[cand.ib[sel]]
        speed[sel] = sp
    span = np.maximum(dt - cand.w0, 0.0)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        q = np.ceil(span * speed / (0.5 * h))
        need = q.astype(np.int64) + 1
    need[speed == 0.0] = MIN_SAMPLES
    count = np.clip(need, MIN_SAMPLES, MAX_SAMPLES)
    count[span == 0.0] = 1
    taus, owner, first = linspace_rows(cand.w0, dt, count)
    wa, wb = _pair_rows(paths, pairs, cand.pair[owner], la, lb, cand.ia[owner], cand.ib[owner], taus)
    d = tri_pair_distance(wa, wb)
    return taus, d, owner, first, count, h, speed


def _zoom_grid(a, b):
    g, _, _ = linspace_rows(np.array([a]), np.array([b]), np.array([ZOOM_SAMPLES]))
    return g


def _isolate(paths, pairs, entries, counter):
    """Certified zoom per refinement entry (ccd.py:242-308)."""
    states = [{"e": e, "pending": [(e[1], e[2])], "bracket": None} for e in entries]
    for _ in range(64):
        work = []
        for si, st in enumerate(states):
            for iv in st["pending"]:
                work.append((si, iv))
            st["pending"] = []
        if not work:
            break
        grids = [_zoom_grid(a, b) for _, (a, b) in work]
        pair_idx = np.repeat([states[si]["e"][0][0] for si, _ in work], ZOOM_SAMPLES)
        ia = np.repeat([states[si]["e"][0][1] for si, _ in work], ZOOM_SAMPLES)
        ib = np.repeat([states[si]["e"][0][2] for si, _ in work], ZOOM_SAMPLES)
        taus = np.concatenate(grids)
        wa, wb = _pair_rows(paths, pairs, pair_idx, 0, 0, ia, ib, taus)
        dist = tri_pair_distance(wa, wb).reshape(len(work), ZOOM_SAMPLES)
        counter[0] += len(taus)
        for (si, _), g, d in zip(work, grids, dist):
            st = states[si]
            if st["bracket"] is not None and g[0] >= st["bracket"][0]:
                continue
            h, spd = st["e"][3], st["e"][4]
            slack = 0.5 * spd * (g[1] - g[0])
            cut = ZOOM_SAMPLES
            hit = np.flatnonzero(d <= h)
            if len(hit):
                j = int(hit[0])
                st["bracket"] = (float(g[j - 1]) if j > 0 else float(g[0]), float(g[j]))
                cut = j
            if slack <= GRAZE_TOL:
                continue
            flag = d[:cut] <= h + slack
            for lo_i, hi_i in _runs(flag):
                sub = (float(g[max(lo_i - 1, 0)]), float(g[min(hi_i + 1, cut - 1)]))
                if sub[1] > sub[0]:
                    st["pending"].append(sub)
    return [(st["e"][0], st["bracket"][0], st["bracket"][1], st["e"][3])
            for st in states if st["bracket"] is not None]


def _runs(flag):
    """Maximal runs [first, last] of True in a 1-D bool array."""
    out = []
    k = 0
    n = len(flag)
    while k < n:
        if not flag[k]:
            k += 1
            continue
        e = k
        while e + 1 < n and flag[e + 1]:
            e += 1
        out.append((k, e))
        k = e + 1
    return out


def _bisect(paths, pairs, brackets, counter):
    """52-step bisection to the first crossing (ccd.py:311-318)."""
    rows = [b[0] for b in brackets]
    pair_idx = np.array([r[0] for r in rows])
    ia = np.array([r[1] for r in rows])
    ib = np.array([r[2] for r in rows])
    lo = np.array([b[1] for b in brackets])
    hi = np.array([b[2] for b in brackets])
    h = np.array([b[3] for b in brackets])
    for _ in range(BISECT_ITERS):
        mid = 0.5 * (lo + hi)
        wa, wb = _pair_rows(paths, pairs, pair_idx, 0, 0, ia, ib, mid)
        below = tri_pair_distance(wa, wb) <= h
        counter[0] += len(mid)
        hi = np.where(below, mid, hi)
        lo = np.where(below, lo, mid)
    return hi


def search(paths, pairs, dt, widen=WIDEN, exhaustive=False) -> SearchOutput:
    """The multiscale earliest-contact search (ccd.py:373-487), raw records."""
    dt = float(dt)
    seeds = {}
    for k, (ba, bb) in enumerate(pairs):
        ta, tb = paths[ba].tree, paths[bb].tree
        la = 0 if exhaustive else len(ta.levels) - 1
        lb = 0 if exhaustive else len(tb.levels) - 1
        na, nb = ta.levels[la].size, tb.levels[lb].size
        ia, ib = np.meshgrid(np.arange(na), np.arange(nb), indexing="ij")
        seeds.setdefault((la, lb), []).append(
            Candidates(np.full(na * nb, k), ia.ravel(), ib.ravel(), np.zeros(na * nb)))
    buckets = {key: _cat(v) for key, v in seeds.items()}
    out = SearchOutput(dt=dt, collision=False, first_contact=None, narrowing_iters=0,
                       bound_history=[])
    entries = []
    while buckets:
        la, lb = max(buckets, key=lambda key: (max(key), key[0] + key[1]))
        cand = buckets.pop((la, lb))
        if not len(cand):
            continue
        taus, d, owner, first, count, h, speed = _screen(paths, pairs, la, lb, cand, dt)
        out.rows += len(taus)
        fine = la == 0 and lb == 0
        step = np.zeros(len(cand))
        multi = count > 1
        step[multi] = taus[first[multi] + 1] - taus[first[multi]]
        thr = h + 0.5 * speed * step
        flag = d <= thr[owner]
        children = {}
        for i in range(len(cand)):
            s0, n_s = int(first[i]), int(count[i])
            di = d[s0:s0 + n_s]
            gi = taus[s0:s0 + n_s]
            k_pair, ia, ib, w0 = int(cand.pair[i]), int(cand.ia[i]), int(cand.ib[i]), cand.w0[i]
            if fine and w0 == 0.0 and di[0] <= h[i] + REST_SLOP:
                out.resting.append((k_pair, ia, ib, float(h[i])))
                continue
            fl = flag[s0:s0 + n_s]
            if not fl.any():
                continue
            if not fine:
                k0 = int(np.argmax(fl))
                w_child = float(gi[max(k0 - 1, 0)])
                pa, pb = paths[pairs[k_pair][0]], paths[pairs[k_pair][1]]
                kids_a = pa.tree.levels[la].children[ia] if la > 0 else np.array([ia])
                kids_b = pb.tree.levels[lb].children[ib] if lb > 0 else np.array([ib])
                key = (la - 1 if la > 0 else 0, lb - 1 if lb > 0 else 0)
                ca, cb = np.meshgrid(np.asarray(kids_a), np.asarray(kids_b), indexing="ij")
                children.setdefault(key, []).append(Candidates(
                    np.full(ca.size, k_pair), ca.ravel().astype(np.int64),
                    cb.ravel().astype(np.int64), np.full(ca.size, w_child)))
                continue
            for r0, r1 in _runs(fl):
                lo_i = max(r0 - 1, 0)
                hi_i = min(r1 + 1, n_s - 1)
                if di[lo_i] <= h[i]:
                    out.crossings.append((float(gi[lo_i]), k_pair, ia, ib, float(h[i])))
                elif hi_i > lo_i:
                    entries.append(((k_pair, ia, ib), float(gi[lo_i]), float(gi[hi_i]),
                                    float(h[i]), float(speed[i])))
        for key, lst in children.items():
            if key in buckets:
                buckets[key] = _cat([buckets[key]] + lst)
            else:
                buckets[key] = _cat(lst)
    bound = dt
    if entries:
        zc = [0]
        brackets = _isolate(paths, pairs, entries, zc)
        out.zoom_rows = zc[0]
        if brackets:
            bc = [0]
            taus = _bisect(paths, pairs, brackets, bc)
            out.bisect_rows = bc[0]
            for tau, b in sorted((float(t), b) for t, b in zip(taus, brackets)):
                if tau > min(bound * (1.0 + widen), dt):
                    continue
                out.crossings.append((tau, b[0][0], b[0][1], b[0][2], b[3]))
                if tau < bound:
                    bound = tau
                    out.narrowing_iters += 1
                    out.bound_history.append(bound)
    out.collision = bound < dt
    out.dt = min(dt, bound * (1.0 + widen)) if out.collision else dt
    out.first_contact = bound if out.collision else None
    return out


def _cat(parts):
    parts = list(parts)
    return Candidates(*(np.concatenate([getattr(p, f) for p in parts])
                        for f in ("pair", "ia", "ib", "w0")))


# --------------------------------------------------------------------------
# contact records and fusion (ccd.py:43-79, 183-213, 527-577)
# --------------------------------------------------------------------------

@dataclass
class Contact:
    body_a: int
    body_b: int
    position: np.ndarray
    normal: np.ndarray
    depth: float
    t: float
    tri_a: int = -1
    tri_b: int = -1
    threshold: float = 0.0


@dataclass
class Result:
    dt: float
    contacts: list
    narrowing_iters: int
    bound_history: list
    collision: bool
    first_contact: float | None = None
    raw: list = field(default_factory=list)   # pre-fusion records
    stats: dict = field(default_factory=dict)


def contact_record(pa: RigidPath, pb: RigidPath, ia, ib, tau, h, t_abs) -> Contact:
    ta = pa.world(0, [ia], [tau])[0]
    tb = pb.world(0, [ib], [tau])[0]
    dist, wa, wb = tri_pair_witness(ta, tb)
    pos = 0.5 * (wa + wb)
    na = unit_face_normal(ta)
    nb = unit_face_normal(tb)
    if abs(float(dot_blas(na, nb))) >= PARALLEL_COS:
        mid = overlap_centroid(ta, tb, na)
        if mid is not None:
            pos = mid
    if dist > 1e-9:
        nrm = (wa - wb) / dist
    else:
        nrm = nb.copy()
        if float(dot_blas(nrm, _mean3(ta) - _mean3(tb))) < 0.0:
            nrm = -nrm
    return Contact(pa.bid, pb.bid, pos, nrm, max(0.0, h - dist), t_abs, int(ia), int(ib), float(h))


def fuse(contacts):
    """filter_contacts (ccd.py:527-577)."""
    groups = {}
    for c in contacts:
        groups.setdefault((c.body_a, c.body_b), []).append(c)
    fused = []
    for key in sorted(groups):
        pts = sorted(groups[key], key=lambda c: (
            c.t, round9(c.position[0]), round9(c.position[1]),
            round9(c.position[2]), c.tri_a, c.tri_b))
        n = len(pts)
        parent = list(range(n))

        def root(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        for i in range(n):
            for j in range(i + 1, n):
                rad = max(pts[i].threshold, pts[j].threshold)
                if float(norm_blas(pts[i].position - pts[j].position)) <= rad:
                    parent[root(j)] = root(i)
        members = {}
        for i in range(n):
            members.setdefault(root(i), []).append(pts[i])
        for r in sorted(members):
            grp = members[r]
            pos = grp[0].position.copy()
            nsum = grp[0].normal.copy()
            for c in grp[1:]:
                pos = pos + c.position
                nsum = nsum + c.normal
            pos = pos / len(grp)
            ln = float(norm_blas(nsum))
            nrm = nsum / ln if ln > 1e-12 else grp[0].normal
            rep = min(grp, key=lambda c: (c.t, -c.depth))
            fused.append(Contact(rep.body_a, rep.body_b, pos, nrm,
                                 max(c.depth for c in grp), min(c.t for c in grp),
                                 rep.tri_a, rep.tri_b, max(c.threshold for c in grp)))
    return fused


def _finish(paths, pairs, so: SearchOutput, t_base) -> Result:
    raw = []
    for k, ia, ib, h in so.resting:
        raw.append(contact_record(paths[pairs[k][0]], paths[pairs[k][1]], ia, ib, 0.0, h, t_base))
    for tau, k, ia, ib, h in so.crossings:
        if tau <= so.dt:
            raw.append(contact_record(paths[pairs[k][0]], paths[pairs[k][1]], ia, ib, tau, h,
                                      t_base + tau))
    return Result(dt=so.dt, contacts=fuse(raw), narrowing_iters=so.narrowing_iters,
                  bound_history=list(so.bound_history), collision=so.collision,
                  first_contact=so.first_contact, raw=raw,
                  stats={"rows": so.rows, "zoom_rows": so.zoom_rows,
                         "bisect_rows": so.bisect_rows})


def pair_earliest_contact(body_a, body_b, dt, *, widen=WIDEN, exhaustive=False) -> Result:
    """ccd.pair_earliest_contact (ccd.py:490-502)."""
    pa, pb = RigidPath(body_a), RigidPath(body_b)
    paths = {pa.bid: pa, pb.bid: pb}
    pairs = [(pa.bid, pb.bid)]
    so = search(paths, pairs, dt, widen, exhaustive)
    return _finish(paths, pairs, so, 0.0)


def compute_effective_dt(cluster, particles, statics, pairs, *, widen=WIDEN) -> Result:
    """ccd.compute_effective_dt (ccd.py:505-524)."""
    pairs = [(int(a), int(b)) for a, b in pairs]
    if not pairs:
        return Result(dt=cluster.dt, contacts=[], narrowing_iters=0, bound_history=[],
                      collision=False)
    paths = {}
    for a, b in pairs:
        for bid in (a, b):
            if bid not in paths:
                paths[bid] = RigidPath(particles[bid] if bid >= 0 else statics[bid])
    so = search(paths, pairs, float(cluster.dt), widen)
    return _finish(paths, pairs, so, cluster.t_current)
