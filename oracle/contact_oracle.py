"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the contact consumers.

A plain-Python/numpy restatement of the reference's contact resolution
(`ltsdem.contacts`, /root/reference/pkg/src/ltsdem/contacts.py), used by
`tests/` as the checker and by `bench.py`'s CPU legs.  The product package
never imports it.

What it restates (file:line under /root/reference/pkg/src/ltsdem):

* `color_contact_graph` (contacts.py:58-78)
* `_Arm.mobility` (:92-97), `_contact_arm` (:100-111), `solve_impulses`
  (:114-198), `_relative_velocity` (:201-204), `_apply` (:207-213),
  `_impulse_measure` (:216-222)
* `integrate_cluster` (:225-253) and `apply_separation` (:256-285), with
  `state.extrapolate_free_flight` (state.py:89-99), `quaternions.advance`
  (quaternions.py:85-90) and `quaternions.to_matrix` (:54-63) for
  `Particle.inverse_inertia_world` (body.py:39-41)

Library-decided roundings (`fpexact.py`): 1-D `@` / `np.linalg.norm` are
OpenBLAS `ddot` FMA chains, `(3,3) @ (3,)` is `dgemv`
(fma(m2,v2, fma(m0,v0, m1*v1))), `(3,3) @ (3,3)` is `dgemm` (an FMA chain
over k), `np.cross` and elementwise numpy are separately rounded, and
`np.mean(axis=0)` over a list of 3-vectors sums the rows in order.  Pinned
by `tests/golden/contacts.npz`, produced by the reference itself
(`tests/golden/make_golden_contacts.py`).

Body records are the layout of include/ltsgpu.h (`ltsg_solve_input`): per
body [0:3] position [3:6] velocity [6:10] rotation [10:13] angular
velocity [13] t [14] inverse mass (1 / mass) [15:24] body-frame inverse
inertia, row-major.
"""

from __future__ import annotations

import numpy as np

from .fpexact import cross3, dot_blas, fma

B_POS, B_VEL, B_ROT, B_OMEGA, B_T, B_INVM, B_INVI = 0, 3, 6, 10, 13, 14, 15
B_RECORD = 24


def _dot(a, b) -> float:
    return float(dot_blas(np.asarray(a), np.asarray(b)))


def _norm(a) -> float:
    return float(np.sqrt(_dot(a, a)))


def _gemv(m, v):
    """(3,3) @ (3,) through OpenBLAS dgemv."""
    return np.array([float(fma(m[i, 2], v[2], fma(m[i, 0], v[0], m[i, 1] * v[1]))) for i in range(3)])


def _gemm(a, b):
    """(3,3) @ (3,3) through OpenBLAS dgemm: an FMA chain over k per entry."""
    out = np.empty((3, 3))
    for i in range(3):
        for j in range(3):
            out[i, j] = float(fma(a[i, 2], b[2, j], fma(a[i, 1], b[1, j], a[i, 0] * b[0, j])))
    return out


def _cross(a, b):
    return cross3(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64))


def _normalize4(q):
    n = float(np.sqrt(fma(q[3], q[3], fma(q[2], q[2], fma(q[1], q[1], q[0] * q[0])))))
    return q / n


def _multiply(p, q):
    w1, x1, y1, z1 = (float(v) for v in p)
    w2, x2, y2, z2 = (float(v) for v in q)
    return np.array([
        w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
        w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
        w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
        w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2,
    ])


def advance(q, omega, dt):
    """quaternions.advance (:85-90) with from_rotation_vector (:75-82)."""
    phi = np.asarray(omega, dtype=np.float64) * dt
    angle = _norm(phi)
    if angle < 1e-12:
        dq = _normalize4(np.concatenate(([1.0], 0.5 * phi)))
    else:
        half = 0.5 * angle
        dq = np.concatenate(([np.cos(half)], np.sin(half) * phi / angle))
    return _normalize4(_multiply(dq, q))


def to_matrix(q):
    """quaternions.to_matrix (:54-63), Python scalar arithmetic."""
    w, x, y, z = (float(v) for v in q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def extrapolate(state, dt):
    """state.extrapolate_free_flight (state.py:89-99) on a (pos, vel, rot, omega, t) tuple."""
    if dt < 0.0:
        raise ValueError(f"free flight requires dt >= 0, got {dt}")
    pos, vel, rot, om, t = state
    return (pos + dt * vel, vel.copy(), advance(rot, om, dt), om.copy(), t + dt)


def _state(rec):
    return (rec[B_POS:B_POS + 3].copy(), rec[B_VEL:B_VEL + 3].copy(), rec[B_ROT:B_ROT + 4].copy(),
            rec[B_OMEGA:B_OMEGA + 3].copy(), float(rec[B_T]))


def color_contact_graph(sides):
    """contacts.py:58-78 on (body_a, body_b) id pairs (negative = static)."""
    classes, used = [], []
    for idx, (a, b) in enumerate(sides):
        bodies = {bid for bid in (a, b) if bid >= 0}
        for k, taken in enumerate(used):
            if not taken & bodies:
                classes[k].append(idx)
                taken |= bodies
                break
        else:
            classes.append([idx])
            used.append(set(bodies))
    return classes


class _Arm:
    __slots__ = ("pid", "inv_mass", "r", "inv_inertia")

    def __init__(self, pid, inv_mass, r, inv_inertia):
        self.pid, self.inv_mass, self.r, self.inv_inertia = pid, inv_mass, r, inv_inertia

    def mobility(self, d):
        if self.inv_mass == 0.0:
            return 0.0
        rxd = _cross(self.r, d)
        return self.inv_mass + _dot(d, _cross(_gemv(self.inv_inertia, rxd), self.r))


def _rel(a, b, vel, ang):
    va = vel[a.pid] + _cross(ang[a.pid], a.r) if a.pid >= 0 else np.zeros(3)
    vb = vel[b.pid] + _cross(ang[b.pid], b.r) if b.pid >= 0 else np.zeros(3)
    return va - vb


def _apply(a, b, imp, vel, ang):
    if a.pid >= 0:
        vel[a.pid] = vel[a.pid] + a.inv_mass * imp
        ang[a.pid] = ang[a.pid] + _gemv(a.inv_inertia, _cross(a.r, imp))
    if b.pid >= 0:
        vel[b.pid] = vel[b.pid] - b.inv_mass * imp
        ang[b.pid] = ang[b.pid] - _gemv(b.inv_inertia, _cross(b.r, imp))


def _measure(a, b, imp):
    m = _norm(imp)
    for side in (a, b):
        if side.pid >= 0:
            m = max(m, _norm(_cross(side.r, imp)))
    return m


def solve_impulses(contacts, bodies, cfg):
    """contacts.py:114-198.  `contacts`: list of dicts with body_a, body_b
    (ids; negative = static), position, normal, t; `bodies`: id -> record.
    `cfg`: restitution, friction, relaxation, penalty, threshold,
    max_iterations.  Returns (velocities, angular_velocities, iterations,
    converged, normal_impulses, friction_impulses)."""
    if not contacts:
        return {}, {}, 0, True, [], []
    vel, ang, arms = {}, {}, []
    k_normal = np.empty(len(contacts))
    bias = np.empty(len(contacts))
    for i, c in enumerate(contacts):
        sides = []
        for bid in (c["body_a"], c["body_b"]):
            if bid < 0:
                sides.append(_Arm(bid, 0.0, np.zeros(3), np.zeros((3, 3))))
                continue
            rec = bodies[bid]
            s0 = _state(rec)
            at = extrapolate(s0, c["t"] - s0[4])
            rot = to_matrix(at[2])
            inv_i = _gemm(_gemm(rot, rec[B_INVI:B_INVI + 9].reshape(3, 3)), rot.T)
            arm = _Arm(bid, float(rec[B_INVM]), None, inv_i)
            com = s0[0] + (c["t"] - s0[4]) * s0[1]
            arm.r = np.asarray(c["position"], dtype=np.float64) - com
            if bid not in vel:
                vel[bid] = s0[1].copy()
                ang[bid] = s0[3].copy()
            sides.append(arm)
        a, b = sides
        arms.append((a, b))
        n = np.asarray(c["normal"], dtype=np.float64)
        k_normal[i] = a.mobility(n) + b.mobility(n)
        vn0 = _dot(_rel(a, b, vel, ang), n)
        bias[i] = -cfg["restitution"] * min(vn0, 0.0)
    classes = color_contact_graph([(c["body_a"], c["body_b"]) for c in contacts])
    lam = np.zeros(len(contacts))
    fric = [np.zeros(3) for _ in contacts]
    iterations, converged = 0, False
    relax, pen, mu = cfg["relaxation"], cfg["penalty"], cfg["friction"]
    while iterations < cfg["max_iterations"] and not converged:
        iterations += 1
        worst = 0.0
        for cls in classes:
            for i in cls:
                a, b = arms[i]
                n = np.asarray(contacts[i]["normal"], dtype=np.float64)
                v_rel = _rel(a, b, vel, ang)
                d_lam = relax * pen * (bias[i] - _dot(v_rel, n)) / k_normal[i]
                new_lam = max(lam[i] + d_lam, 0.0)
                applied = (new_lam - lam[i]) * n
                lam[i] = new_lam
                _apply(a, b, applied, vel, ang)
                worst = max(worst, _measure(a, b, applied))
                if mu > 0.0 and lam[i] > 0.0:
                    v_rel = _rel(a, b, vel, ang)
                    vt = v_rel - _dot(v_rel, n) * n
                    speed = _norm(vt)
                    if speed > 1e-12:
                        t_dir = vt / speed
                        k_t = a.mobility(t_dir) + b.mobility(t_dir)
                        target = fric[i] - (relax * speed / k_t) * t_dir
                        cap = mu * lam[i]
                        scale = _norm(target)
                        if scale > cap:
                            target = target * (cap / scale)
                        applied = target - fric[i]
                        fric[i] = target
                        _apply(a, b, applied, vel, ang)
                        worst = max(worst, _measure(a, b, applied))
        converged = worst < cfg["threshold"]
    return vel, ang, iterations, converged, [float(x) for x in lam], fric


def integrate_cluster(members, t_new, contacts, bodies, solution):
    """contacts.py:225-253: the prospective new snapshot of every member, as
    (pos, vel, rot, omega, t) tuples keyed by id."""
    first = {}
    for c in contacts:
        for bid in (c["body_a"], c["body_b"]):
            if bid >= 0:
                t = first.get(bid)
                first[bid] = c["t"] if t is None else min(t, c["t"])
    out = {}
    for pid in members:
        s0 = _state(bodies[pid])
        t_c = first.get(pid)
        if t_c is None or solution is None or pid not in solution[0]:
            out[pid] = extrapolate(s0, t_new - s0[4])
        else:
            pre = extrapolate(s0, t_c - s0[4])
            pre = (pre[0], solution[0][pid].copy(), pre[2], solution[1][pid].copy(), pre[4])
            out[pid] = extrapolate(pre, t_new - pre[4])
    return out


def apply_separation(contacts, new_states, inv_mass, beta):
    """contacts.py:256-285 on the new snapshots (id -> state tuple, updated in
    place); inv_mass: id -> 1 / mass of the dynamic bodies."""
    pushes = {}
    for c in contacts:
        if c["depth"] > 0.0:
            pushes.setdefault((c["body_a"], c["body_b"]), []).append(c["depth"] * np.asarray(c["normal"]))
    for (a, b), vecs in sorted(pushes.items()):
        wa = inv_mass[a] if a >= 0 else 0.0
        wb = inv_mass[b] if b >= 0 else 0.0
        total = wa + wb
        if total == 0.0:
            continue
        acc = vecs[0].copy()
        for v in vecs[1:]:
            acc = acc + v
        push = beta * (acc / len(vecs))
        if a >= 0 and a in new_states:
            s = new_states[a]
            new_states[a] = (s[0] + push * (wa / total),) + s[1:]
        if b >= 0 and b in new_states:
            s = new_states[b]
            new_states[b] = (s[0] - push * (wb / total),) + s[1:]
    return new_states
