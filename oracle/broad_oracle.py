"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the space-time broad phase.

A numpy restatement of the reference broad phase (`ltsdem.broadphase`,
/root/reference/pkg/src/ltsdem/broadphase.py), used by `tests/` and by
`bench.py`'s CPU legs as the checker and CPU baseline.  The product package
never imports it.

What it restates (file:line under /root/reference/pkg/src/ltsdem):

* `particle_dt` (broadphase.py:46-50) and `pair_window` (:53-56)
* `_Trajectory.of_particle` / `of_static` / `at` / `box` (:73-118), with
  `state.extrapolate_free_flight` (state.py:89-99), `quaternions.advance`
  (quaternions.py:85-90) and `quaternions.rotate` (:42-51) for the sphere
  centre `Particle.sphere_center_at` (body.py:36-37)
* Check 1 `check_spacetime_aabb` (:121-125) and Check 2
  `check_spacetime_tube` / `_min_distance_over_window` (:128-158)
* `build_collision_graph` (:198-252).  The spatial hash `_hash_candidates`
  (:161-195) is "an acceleration only, never a filter": every pair whose
  boxes overlap shares a hash cell, so the result equals the exhaustive
  pair set filtered by Check 1.  The oracle therefore tests all pairs
  (vectorised) and keeps the reference's ordering: edges in sorted
  (index_a, index_b) order over `ids = sorted(pids) + sorted(sids)`,
  static links per particle as sorted tuples, particles in id order.

Library-decided roundings (`fpexact.py`): 1-D `@` and `np.linalg.norm` are
OpenBLAS `ddot` FMA chains; `np.cross` and elementwise numpy are separately
rounded.  Pinned by `tests/golden/broadphase.npz`, produced by the
reference itself (`tests/golden/make_golden_broad.py`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fpexact import cross3, dot_blas, fma

# record layout shared with the product's packing (paper_2309_15417_b200/broadphase.py)
P_OLD_POS, P_OLD_ROT, P_OLD_T = 0, 3, 7
P_CUR_POS, P_CUR_ROT, P_CUR_T = 8, 11, 15
P_VEL, P_OMEGA, P_CENTRE, P_RADIUS = 16, 19, 22, 25
P_RECORD = 28


@dataclass
class Graph:
    edges: dict = field(default_factory=dict)
    static_links: dict = field(default_factory=dict)
    dts: dict = field(default_factory=dict)


# ---------------------------------------------------------------- quaternions

def _dot4(a, b):
    """OpenBLAS ddot for n=4: the FMA chain continued (quaternions.normalize)."""
    return fma(a[..., 3], b[..., 3], fma(a[..., 2], b[..., 2], fma(a[..., 1], b[..., 1], a[..., 0] * b[..., 0])))


def _normalize4(q):
    return q / np.sqrt(_dot4(q, q))[..., None]


def _multiply(q1, q2):
    """quaternions.multiply (quaternions.py:24-35), left to right."""
    w1, x1, y1, z1 = (q1[..., k] for k in range(4))
    w2, x2, y2, z2 = (q2[..., k] for k in range(4))
    return np.stack([
        w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
        w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
        w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
        w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2,
    ], axis=-1)


def advance(q, omega, dt):
    """quaternions.advance (quaternions.py:85-90) row-wise: from_rotation_vector
    (:75-82) of omega*dt, then normalize(multiply(dq, q))."""
    phi = omega * dt[..., None]
    angle = np.sqrt(dot_blas(phi, phi))
    small = angle < 1e-12
    dq_small = _normalize4(np.concatenate([np.ones(phi.shape[:-1] + (1,)), 0.5 * phi], axis=-1))
    half = 0.5 * angle
    with np.errstate(invalid="ignore", divide="ignore"):
        axis = (np.sin(half)[..., None] * phi) / angle[..., None]  # from_axis_angle, n = |phi|
    dq_big = np.concatenate([np.cos(half)[..., None], axis], axis=-1)
    dq = np.where(small[..., None], dq_small, dq_big)
    return _normalize4(_multiply(dq, q))


def rotate(q, v):
    """quaternions.rotate (quaternions.py:42-51): v + 2 (w (u x v) + u x (u x v))."""
    w = q[..., 0:1]
    u = q[..., 1:4]
    uv = cross3(u, v)
    return v + 2.0 * (w * uv + cross3(u, uv))


# ---------------------------------------------------------------- trajectories

def particle_dt(rec, dt_max, growth):
    """broadphase.particle_dt (:46-50) per particle record."""
    last = rec[:, P_CUR_T] - rec[:, P_OLD_T]
    capped = np.minimum(growth * last, dt_max)
    return np.where(last == 0.0, dt_max, capped)


def trajectories(rec, srec, dt):
    """_Trajectory.of_particle / of_static (:83-99): times (n,3), centres
    (n,3,3), radius, ntimes.  Statics carry one knot at t = 0."""
    n_p, n_s = len(rec), len(srec)
    cur_pos = rec[:, P_CUR_POS:P_CUR_POS + 3]
    vel = rec[:, P_VEL:P_VEL + 3]
    centre = rec[:, P_CENTRE:P_CENTRE + 3]
    ext_pos = cur_pos + dt[:, None] * vel                                        # state.py:94
    ext_rot = advance(rec[:, P_CUR_ROT:P_CUR_ROT + 4], rec[:, P_OMEGA:P_OMEGA + 3], dt)
    c_old = rec[:, P_OLD_POS:P_OLD_POS + 3] + rotate(rec[:, P_OLD_ROT:P_OLD_ROT + 4], centre)
    c_cur = cur_pos + rotate(rec[:, P_CUR_ROT:P_CUR_ROT + 4], centre)
    c_ext = ext_pos + rotate(ext_rot, centre)
    times = np.zeros((n_p + n_s, 3))
    times[:n_p, 0] = rec[:, P_OLD_T]
    times[:n_p, 1] = rec[:, P_CUR_T]
    times[:n_p, 2] = rec[:, P_CUR_T] + dt
    centres = np.zeros((n_p + n_s, 3, 3))
    centres[:n_p] = np.stack([c_old, c_cur, c_ext], axis=1)
    centres[n_p:] = srec[:, None, 0:3]
    radius = np.concatenate([rec[:, P_RADIUS], srec[:, 3]])
    ntimes = np.concatenate([np.full(n_p, 3), np.ones(n_s, dtype=np.int64)])
    return times, centres, radius, ntimes


def boxes(centres, radius, ntimes):
    """_Trajectory.box (:115-118)."""
    c = np.where((ntimes == 1)[:, None, None], centres[:, :1, :], centres)
    return c.min(axis=1) - radius[:, None], c.max(axis=1) + radius[:, None]


def _at(times, centres, ntimes, t):
    """_Trajectory.at (:101-113) row-wise."""
    t = np.minimum(np.maximum(t, times[:, 0]), times[:, 2])
    first = t <= times[:, 1]
    a = np.where(first[:, None], centres[:, 0], centres[:, 1])
    b = np.where(first[:, None], centres[:, 1], centres[:, 2])
    ta = np.where(first, times[:, 0], times[:, 1])
    tb = np.where(first, times[:, 1], times[:, 2])
    span = tb - ta
    with np.errstate(invalid="ignore", divide="ignore"):
        u = (t - ta) / span
    moved = (1.0 - u)[:, None] * a + u[:, None] * b
    out = np.where((span == 0.0)[:, None], b, moved)
    return np.where((ntimes == 1)[:, None], centres[:, 0], out)


def min_distance(t1, c1, n1, t2, c2, n2, w0, w1):
    """_min_distance_over_window (:128-151) for rows of trajectory pairs."""
    m = len(w0)
    best = np.full(m, np.inf)
    if m == 0:
        return best
    inside = []
    for tt, nn in ((t1, n1), (t2, n2)):
        for k in range(3):
            v = tt[:, k]
            ok = (k < nn) & (w0 < v) & (v < w1)
            inside.append(np.where(ok, v, np.inf))
    knots = np.sort(np.stack([w0, w1] + inside, axis=1), axis=1)
    dup = np.zeros_like(knots, dtype=bool)
    dup[:, 1:] = knots[:, 1:] == knots[:, :-1]          # the reference's knot set
    knots = np.sort(np.where(dup, np.inf, knots), axis=1)
    count = np.isfinite(knots).sum(axis=1)
    for k in range(knots.shape[1] - 1):
        live = (k + 1 < count) & (w1 >= w0)
        if not live.any():
            continue
        ta = np.where(live, knots[:, k], w0)
        tb = np.where(live, knots[:, k + 1], w0)
        d0 = _at(t1, c1, n1, ta) - _at(t2, c2, n2, ta)
        d1 = _at(t1, c1, n1, tb) - _at(t2, c2, n2, tb)
        dd = d1 - d0
        denom = dot_blas(dd, dd)
        with np.errstate(invalid="ignore", divide="ignore"):
            s = np.clip(-dot_blas(d0, dd) / denom, 0.0, 1.0)
        s = np.where(denom == 0.0, 0.0, s)
        v = d0 + s[:, None] * dd
        d = np.sqrt(dot_blas(v, v))
        best = np.where(live & (d < best), d, best)
    single = (count == 1) & (w1 >= w0)
    if single.any():
        d = _at(t1, c1, n1, w0) - _at(t2, c2, n2, w0)
        best = np.where(single, np.sqrt(dot_blas(d, d)), best)
    return best


def build_collision_graph(rec, srec, pids, sids, dt_max, growth=2.0):
    """broadphase.build_collision_graph (:198-252) on packed records
    (rec: (n_p, 28) particle records in ascending pid order; srec: (n_s, 4)
    static world spheres in ascending sid order)."""
    rec = np.asarray(rec, dtype=np.float64).reshape(-1, P_RECORD)
    srec = np.asarray(srec, dtype=np.float64).reshape(-1, 4)
    n_p, n_s = len(rec), len(srec)
    dt = particle_dt(rec, dt_max, growth)
    g = Graph(dts={int(p): float(d) for p, d in zip(pids, dt)})
    times, centres, radius, ntimes = trajectories(rec, srec, dt)
    lo, hi = boxes(centres, radius, ntimes)
    n = n_p + n_s
    # Check 1 over every pair (i < j, i a particle: two statics never meet,
    # :228-229), in row blocks to bound memory; (i, j) stays in sorted order
    I, J = [], []
    step = max(1, (1 << 22) // max(n, 1))
    for i0 in range(0, n_p, step):
        i1 = min(n_p, i0 + step)
        ii = np.repeat(np.arange(i0, i1), n)
        jj = np.tile(np.arange(n), i1 - i0)
        keep = jj > ii
        ii, jj = ii[keep], jj[keep]
        ov = np.all(lo[ii] <= hi[jj], axis=1) & np.all(lo[jj] <= hi[ii], axis=1)
        I.append(ii[ov])
        J.append(jj[ov])
    ii = np.concatenate(I) if I else np.zeros(0, dtype=np.int64)
    jj = np.concatenate(J) if J else np.zeros(0, dtype=np.int64)
    dyn = jj < n_p
    cur_t = rec[:, P_CUR_T]
    # pair_window (:53-56) for two particles; (old.t, t_cur + dt) against a static
    ta_, tb_ = cur_t[ii], np.where(dyn, cur_t[np.minimum(jj, n_p - 1)], 0.0)
    da, db = dt[ii], np.where(dyn, dt[np.minimum(jj, n_p - 1)], 0.0)
    start = np.minimum(ta_, tb_)
    w0 = np.where(dyn, start, rec[ii, P_OLD_T])
    w1 = np.where(dyn, start + np.minimum(da, db), cur_t[ii] + dt[ii])
    best = min_distance(times[ii], centres[ii], ntimes[ii], times[jj], centres[jj], ntimes[jj], w0, w1)
    hit = best <= radius[ii] + radius[jj]                 # Check 2
    links: dict = {}
    for i, j, a, b, h, d in zip(ii, jj, w0, w1, hit, dyn):
        if not h:
            continue
        if d:
            g.edges[(int(pids[i]), int(pids[j]))] = (float(a), float(b))
        else:
            links.setdefault(int(pids[i]), []).append(int(sids[j - n_p]))
    g.static_links = {p: tuple(sorted(set(v))) for p, v in links.items()}
    g.candidates = int(len(ii))
    return g


def tube_rows(t1, c1, r1, t2, c2, r2, w0, w1, n1=None, n2=None):
    """check_spacetime_tube (:154-158) for rows of explicit trajectories."""
    n1 = np.full(len(w0), 3) if n1 is None else n1
    n2 = np.full(len(w0), 3) if n2 is None else n2
    best = min_distance(t1, c1, n1, t2, c2, n2, w0, w1)
    return best, best <= r1 + r2
