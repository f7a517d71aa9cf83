"""Generate the golden fixtures by running the REFERENCE (ltsdem) itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py [--quick]

Outputs (all small, committed):
  kernels.npz   point-triangle / segment-segment / 15-feature rows and outputs
  witness.npz   _closest_feature witness points, face normals, overlap centroids
  fusion.npz    filter_contacts inputs and outputs
  trees.npz     meshes and reference-built surrogate trees
  scenes_ccd.npz       the reference's own test_ccd.py known-answer scenes
  scenes_crit2.npz     acceptance criterion 2's 200 seeded pairs (replayed)
  scenes_configs.npz   small c1..c5-shaped scenes (reference-built trees)
  engine_sweeps.npz    the reference engine's sweeps on its "pairs" scenario:
                       every cluster's cache key, result and cache hit/miss
  scenes_baseline.npz  c4 pairs and c5 clusters drawn from the bench workloads
                       at their BASELINE shapes (1280-tri spinning pairs;
                       20480-tri icospheres against 12-tri boxes)

Each scene records the reference result, the raw (pre-fusion) contact list
(captured by wrapping ccd.filter_contacts, which _search resolves as a
module global at call time, ccd.py:482) and the total number of
_feature_distances rows (screen + zoom + bisection).

Fixture inputs are seeded; the reference runs on them unmodified.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from ltsdem import ccd, kernels, quaternions  # noqa: E402
from ltsdem.body import initial_state, make_particle, make_static  # noqa: E402
from ltsdem.clustering import Cluster  # noqa: E402
from ltsdem.mesh import TriangleMesh, make_cube, make_noisy_sphere, make_plane  # noqa: E402
from ltsdem.surrogate import build_surrogate_tree  # noqa: E402

import gio  # noqa: E402
import scene_codec as SC  # noqa: E402
from paper_2309_15417_b200 import scenes as S  # noqa: E402


# ------------------------------------------------------------------ helpers

class Recorder:
    """Wrap ccd.filter_contacts / ccd._feature_distances for one call."""

    def __enter__(self):
        self.raw = []
        self.rows = 0
        self._f, self._d = ccd.filter_contacts, ccd._feature_distances
        rec = self

        def filt(cs):
            rec.raw.extend(cs)
            return rec._f(cs)

        def dist(a, b):
            rec.rows += len(a)
            return rec._d(a, b)

        ccd.filter_contacts = filt
        ccd._feature_distances = dist
        return self

    def __exit__(self, *exc):
        ccd.filter_contacts, ccd._feature_distances = self._f, self._d


def pair_case(name, a, b, dt, exhaustive=False, widen=1e-3, dedup=False):
    with Recorder() as r:
        res = ccd.pair_earliest_contact(a, b, dt, widen=widen, exhaustive=exhaustive)
    return {"name": name, "mode": "pair", "bodies": [SC.encode_body(a, dedup), SC.encode_body(b, dedup)],
            "pairs": np.array([[_bid(a), _bid(b)]], dtype=np.int64), "dt": float(dt),
            "widen": float(widen), "exhaustive": bool(exhaustive), "t_base": 0.0,
            "result": SC.encode_result(res, r.raw), "rows": int(r.rows)}


def cluster_case(name, cluster, particles, statics, pairs, widen=1e-3, dedup=False):
    with Recorder() as r:
        res = ccd.compute_effective_dt(cluster, particles, statics, pairs, widen=widen)
    bodies = [SC.encode_body(p, dedup) for p in particles.values()] + \
             [SC.encode_body(s, dedup) for s in statics.values()]
    return {"name": name, "mode": "cluster", "bodies": bodies,
            "pairs": np.array(list(pairs), dtype=np.int64).reshape(-1, 2),
            "dt": float(cluster.dt), "widen": float(widen), "exhaustive": False,
            "t_base": float(cluster.t_current),
            "result": SC.encode_result(res, r.raw), "rows": int(r.rows)}


def _bid(body):
    return body.pid if hasattr(body, "timeline") else body.sid


def ref_particle(pid, v, f, eps, **state):
    return make_particle(pid, TriangleMesh(v, f), eps, initial_state(**state))


# ------------------------------------------------------------------ kernels

def gen_kernels(rng):
    n = 3000
    # point-triangle: random, plus points steered into each Voronoi region
    p, a, b, c = (rng.normal(size=(n, 3)) for _ in range(4))
    tri = rng.normal(size=(600, 3, 3))
    bary = rng.dirichlet((1, 1, 1), size=600)
    face_pts = np.einsum("ni,nij->nj", bary, tri)
    nrm = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    face_pts = face_pts + nrm * rng.normal(size=(600, 1))
    edge_pts = tri[:, 0] + rng.uniform(-0.2, 1.2, (600, 1)) * (tri[:, 1] - tri[:, 0]) \
        + 0.3 * rng.normal(size=(600, 3))
    degen = rng.normal(size=(200, 3, 3))
    degen[:100, 2] = degen[:100, 0] + rng.uniform(-2, 2, (100, 1)) * (degen[:100, 1] - degen[:100, 0])
    degen[100:, 1] = degen[100:, 0]
    degen[150:, 2] = degen[150:, 0]
    exact = np.array([[0.0, 0, 0], [2, 0, 0], [0, 2, 0]])
    known_p = np.array([[0.4, 0.4, 1.5], [-1.0, -1.0, 0.0], [0.5, -1.0, 0.0], [3.0, 3.0, 0.0],
                        [1.0, 1.0, 0.0], [0.0, 0.0, 0.0]])
    P = np.concatenate([p, face_pts, edge_pts, rng.normal(size=(200, 3)), known_p])
    A = np.concatenate([a, tri[:, 0], tri[:, 0], degen[:, 0], np.repeat(exact[None, 0], 6, 0)])
    Bv = np.concatenate([b, tri[:, 1], tri[:, 1], degen[:, 1], np.repeat(exact[None, 1], 6, 0)])
    C = np.concatenate([c, tri[:, 2], tri[:, 2], degen[:, 2], np.repeat(exact[None, 2], 6, 0)])
    scale = rng.choice([1.0, 1e-3, 1e3], size=(len(P), 1))
    P, A, Bv, C = P * scale, A * scale, Bv * scale, C * scale
    pt_d, pt_c = kernels.point_triangle_closest(P, A, Bv, C)

    # segment-segment: random, parallel, collinear, degenerate
    p1, q1, p2, q2 = (rng.normal(size=(n, 3)) for _ in range(4))
    m = 300
    d = rng.normal(size=(m, 3))
    par = [rng.normal(size=(m, 3)), None, rng.normal(size=(m, 3)), None]
    par[1] = par[0] + d * rng.uniform(0.1, 2, (m, 1))
    par[3] = par[2] + d * rng.uniform(-2, 2, (m, 1))
    col = [rng.normal(size=(m, 3)), None, None, None]
    col[1] = col[0] + d
    col[2] = col[0] + d * rng.uniform(-1, 2, (m, 1))
    col[3] = col[0] + d * rng.uniform(-1, 2, (m, 1))
    dg = [rng.normal(size=(m, 3)) for _ in range(4)]
    dg[1][: m // 2] = dg[0][: m // 2]
    dg[3][m // 3:] = dg[2][m // 3:]
    known = [np.array([[-1.0, 0, 0], [0, 0, 0], [0, 0, 0]]), np.array([[1.0, 0, 0], [1, 0, 0], [0, 0, 0]]),
             np.array([[0.0, -1, 1], [0, 1, 0], [3, 4, 0]]), np.array([[0.0, 1, 1], [1, 1, 0], [3, 4, 0]])]
    segs = [np.concatenate([x, y, z, w, k]) for x, y, z, w, k in zip(
        (p1, q1, p2, q2), par, col, dg, known)]
    scale = rng.choice([1.0, 1e-3, 1e3], size=(len(segs[0]), 1))
    segs = [s * scale for s in segs]
    ss_d, ss_c1, ss_c2 = kernels.segment_segment_closest(*segs)

    # 15-feature rows: random pairs, near pairs at several scales, mesh-derived rows
    k = 4000
    ta = rng.normal(size=(k, 3, 3))
    tb = rng.normal(size=(k, 3, 3))
    near_a = rng.normal(size=(k, 3, 3)) * 0.1
    near_b = near_a[:, [1, 2, 0]] + rng.normal(size=(k, 1, 3)) * 0.05 + rng.normal(size=(k, 3, 3)) * 0.05
    s = rng.choice([1.0, 1e-2, 1e2], size=(k, 1, 1))
    v0, f = S.icosphere(2)
    va = v0 * (1 + rng.uniform(-0.05, 0.05, len(v0)))[:, None]
    vb = v0 * (1 + rng.uniform(-0.05, 0.05, len(v0)))[:, None] + np.array([2.02, 0.0, 0.0])
    ca = np.stack([va[f[:, 0]], va[f[:, 1]], va[f[:, 2]]], 1)
    cb = np.stack([vb[f[:, 0]], vb[f[:, 1]], vb[f[:, 2]]], 1)
    ia = rng.integers(0, len(f), 4000)
    ib = rng.integers(0, len(f), 4000)
    FA = np.concatenate([ta, near_a * s, ca[ia]])
    FB = np.concatenate([tb, near_b * s, cb[ib]])
    fd = ccd._feature_distances(FA, FB)
    return {"pt": {"p": P, "a": A, "b": Bv, "c": C, "dist": pt_d, "closest": pt_c},
            "ss": {"p1": segs[0], "q1": segs[1], "p2": segs[2], "q2": segs[3], "dist": ss_d,
                   "c1": ss_c1, "c2": ss_c2},
            "feat": {"ta": FA, "tb": FB, "dist": fd}}


def gen_witness(rng):
    k = 600
    ta = rng.normal(size=(k, 3, 3)) * 0.2
    tb = ta[:, [2, 0, 1]] + rng.normal(size=(k, 1, 3)) * 0.05 + rng.normal(size=(k, 3, 3)) * 0.03
    tb[:100] = ta[:100] + rng.normal(size=(100, 1, 3)) * 1e-12   # coincident -> tiny dist
    dist, pa, pb = [], [], []
    na, nb = [], []
    for x, y in zip(ta, tb):
        d_, a_, b_ = ccd._closest_feature(x, y)
        dist.append(d_)
        pa.append(a_)
        pb.append(b_)
        na.append(ccd._face_normal(x))
        nb.append(ccd._face_normal(y))
    # near-parallel pairs for the overlap centroid
    m = 300
    base = rng.normal(size=(m, 3, 3))
    base[:, :, 2] *= 0.0
    ra = base + rng.normal(size=(m, 1, 3)) * np.array([0.3, 0.3, 0.0])
    rb = base[:, [0, 2, 1]] * rng.uniform(0.5, 1.5, (m, 1, 1)) + np.array([0.0, 0.0, 0.01])
    rb = rb + rng.normal(size=(m, 3, 3)) * np.array([0.2, 0.2, 1e-4])
    q = S.random_quaternions(rng, m)
    cen, has = [], []
    for i in range(m):
        R = quaternions.to_matrix(q[i])
        A_ = ra[i] @ R.T
        B_ = rb[i] @ R.T
        ra[i], rb[i] = A_, B_
        n_ = ccd._face_normal(A_)
        out = kernels.triangle_overlap_centroid(A_, B_, n_)
        has.append(out is not None)
        cen.append(np.zeros(3) if out is None else out)
    return {"ta": ta, "tb": tb, "dist": np.array(dist), "pa": np.array(pa), "pb": np.array(pb),
            "na": np.array(na), "nb": np.array(nb),
            "ov_a": ra, "ov_b": rb, "ov_has": np.array(has), "ov_centroid": np.array(cen)}


def gen_fusion(rng):
    cases = []
    for i in range(40):
        n = int(rng.integers(1, 60))
        pairs = [(0, 1), (0, 2), (3, -1), (1, 2)][: int(rng.integers(1, 5))]
        raw = []
        for _ in range(n):
            ba, bb = pairs[int(rng.integers(len(pairs)))]
            pos = rng.normal(scale=0.02 if i % 2 else 0.3, size=3)
            if raw and rng.uniform() < 0.2:
                pos = raw[int(rng.integers(len(raw)))].position.copy()
            nrm = rng.normal(size=3)
            nrm /= np.linalg.norm(nrm)
            if rng.uniform() < 0.1 and raw:
                nrm = -raw[-1].normal
            raw.append(ccd.ContactPoint(
                body_a=ba, body_b=bb, position=pos, normal=nrm,
                depth=float(rng.choice([0.0, rng.uniform(0, 0.01)])),
                t=float(rng.choice([0.0, 0.5, rng.uniform()])),
                tri_a=int(rng.integers(-1, 50)), tri_b=int(rng.integers(-1, 50)),
                threshold=float(rng.choice([0.02, 0.002, 0.05]))))
        fused = ccd.filter_contacts(list(raw))
        cases.append({"raw": SC.encode_contacts(raw), "fused": SC.encode_contacts(fused)})
    return {"cases": cases}


def gen_trees(rng):
    out = []
    for sub in (0, 1, 2, 3):
        v, f = S.icosphere(sub)
        v = v * (1 + rng.uniform(-0.05, 0.05, len(v)))[:, None]
        t = build_surrogate_tree(TriangleMesh(v, f), 0.01)
        out.append({"vertices": v, "triangles": f, "epsilon": 0.01, "tree": SC.encode_tree(t)})
    for _ in range(3):
        v, f = S.rock(rng)
        t = build_surrogate_tree(TriangleMesh(v * 2.0, f), 0.005)
        out.append({"vertices": v * 2.0, "triangles": f, "epsilon": 0.005, "tree": SC.encode_tree(t)})
    m = make_noisy_sphere(1.0, 48, eta_r=1.2, seed=3)
    t = build_surrogate_tree(m, 0.01)
    out.append({"vertices": m.vertices, "triangles": m.triangles, "epsilon": 0.01,
                "tree": SC.encode_tree(t)})
    return {"trees": out}


# ------------------------------------------------------------------ scenes

def gen_scenes_ccd():
    import test_ccd as T

    cases = []
    a = T._cube(0, (-2.0, 0.0, 0.0), velocity=(1.0, 0.0, 0.0))
    b = T._cube(1, (2.0, 0.0, 0.0), velocity=(-1.0, 0.0, 0.0))
    cases.append(pair_case("head_on_cubes", a, b, 5.0))
    qa = quaternions.from_axis_angle(np.array([0.0, 1.0, 0.0]), np.pi / 4)
    qb = quaternions.from_axis_angle(np.array([1.0, 0.0, 0.0]), np.pi / 4)
    a = T._cube(0, (0.0, 0.0, 2.0), velocity=(0.0, 0.0, -1.0), rotation=qa)
    b = T._cube(1, (0.0, 0.0, 0.0), rotation=qb)
    cases.append(pair_case("crossed_ridges", a, b, 3.0))
    a = T._cube(0, (0.0, 0.0, 1.0 + 1.8 * T.EPS))
    b = T._cube(1, (0.0, 0.0, 0.0))
    cases.append(pair_case("resting_cubes", a, b, 0.8))
    for gap, speed in ((0.1, 0.5), (0.75, 1.0), (2.5, 4.0)):
        a = T._cube(0, (0.0, 0.0, 1.0 + gap), velocity=(0.0, 0.0, -speed))
        b = T._cube(1, (0.0, 0.0, 0.0))
        expected = (gap - T.TOUCH) / speed
        cases.append(pair_case(f"gap_{gap}_{speed}", a, b, 10.0))
        cases.append(pair_case(f"gap_{gap}_{speed}_short", a, b, expected * 0.5))
    a = T._cube(0, (-2.0, 0.0, 0.1), velocity=(1.0, 0.0, 0.0), omega=(0.0, 0.3, 0.0))
    b = T._cube(1, (2.0, 0.0, 0.0), velocity=(-1.0, 0.0, 0.0))
    cases.append(pair_case("spinning_cube", a, b, 5.0))
    rng = np.random.default_rng(5)
    for i in range(10):
        a, b = T._random_pair(rng)
        cases.append(pair_case(f"random_pair_{i}", a, b, 3.0))
        cases.append(pair_case(f"random_pair_{i}_exhaustive", a, b, 3.0, exhaustive=True))
    a = T._cube(0, (-2.0, 0.0, 0.0), velocity=(1.0, 0.0, 0.0))
    b = T._cube(1, (2.0, 0.0, 0.0), velocity=(-1.0, 0.0, 0.0))
    for p in (a, b):
        p.timeline.current.t = 5.0
        p.timeline.old.t = 5.0
    cases.append(cluster_case("cluster_pair", Cluster(members=(0, 1), t_current=5.0, dt=4.0),
                              {0: a, 1: b}, {}, [(0, 1)]))
    floor = make_static(-1, make_plane((-5.0, -5.0, 0.0), (5.0, 5.0, 0.0)), epsilon=T.EPS)
    p = T._cube(0, (0.0, 0.0, 1.0), velocity=(0.0, 0.0, -1.0))
    cases.append(cluster_case("static_floor", Cluster(members=(0,), t_current=0.0, dt=2.0,
                                                      statics=(-1,)), {0: p}, {-1: floor}, [(0, -1)]))
    center = T._cube(0, (0.0, 0.0, 0.0))
    left = T._cube(1, (-3.0, 0.0, 0.0), velocity=(1.0, 0.0, 0.0))
    right = T._cube(2, (3.0, 0.0, 0.0), velocity=(-1.0, 0.0, 0.0))
    cases.append(cluster_case("symmetric_impacts", Cluster(members=(0, 1, 2), t_current=0.0, dt=5.0),
                              {0: center, 1: left, 2: right}, {}, [(0, 1), (0, 2)]))
    # spheres resting on a tilted floor plus a falling cube in one cluster
    s0 = T._sphere(0, (0.0, 0.0, 1.015), n_tris=48)
    s1 = T._sphere(1, (2.5, 0.0, 1.2), velocity=(-0.5, 0.0, -0.4), n_tris=80, omega=(0.2, 0.5, 0.1))
    c2 = T._cube(2, (1.2, 0.1, 3.0), velocity=(0.0, 0.0, -2.0), omega=(1.0, 0.0, 0.3))
    floor = make_static(-1, make_plane((-6.0, -6.0, 0.0), (6.0, 6.0, 0.0)), epsilon=T.EPS)
    cases.append(cluster_case("mixed_cluster", Cluster(members=(0, 1, 2), t_current=1.5, dt=1.0),
                              {0: s0, 1: s1, 2: c2}, {-1: floor},
                              [(0, 1), (0, 2), (1, 2), (0, -1), (1, -1), (2, -1)]))
    return {"cases": cases}


def gen_scenes_crit2(n_exhaustive=30, limit=200):
    import test_acceptance as TA

    rng = np.random.default_rng(20240817)
    plan = ([("hit", 12, 24)] * 45 + [("hit", 32, 48)] * 12 + [("graze", 4, 24)] * 40
            + [("miss", 4, 24)] * 88 + [("rest", 12, 24)] * 5 + [("graze", 26, 48)] * 4
            + [("miss", 26, 48)] * 4 + [("hit", 64, 96)] * 1 + [("miss", 64, 96)] * 1)
    cases = []
    for i, (kind, lo, hi) in enumerate(plan):
        if kind in ("hit", "rest"):
            eta_hi = 1.04 if hi <= 24 else (1.02 if hi <= 48 else 1.01)
        else:
            eta_hi = 1.25 if hi <= 24 else 1.1
        a, b = TA._spawn_pair(rng, TA._pair_mesh(rng, lo, hi, eta_hi),
                              TA._pair_mesh(rng, lo, hi, eta_hi), kind)
        if i >= limit:
            break
        case = pair_case(f"crit2_{i}_{kind}", a, b, TA._C2_DT)
        if i < n_exhaustive:
            ex = pair_case(f"crit2_{i}_{kind}_exhaustive", a, b, TA._C2_DT, exhaustive=True)
            case["exhaustive_result"] = ex["result"]
            case["exhaustive_rows"] = ex["rows"]
        cases.append(case)
    return {"cases": cases}


def gen_scenes_configs(rng):
    cases = []
    # c1-shaped: static noisy icosphere pairs
    for k, sub in enumerate((2, 2, 2, 3)):
        v0, f = S.icosphere(sub)
        va = v0 * (1 + rng.uniform(-0.05, 0.05, len(v0)))[:, None]
        vb = v0 * (1 + rng.uniform(-0.05, 0.05, len(v0)))[:, None]
        q = S.random_quaternions(rng, 2)
        d = rng.uniform(1.9, 2.1)
        ax = S.unit_vectors(rng, 1)[0]
        a = ref_particle(0, va, f, 0.01, position=-0.5 * d * ax, rotation=q[0])
        b = ref_particle(1, vb, f, 0.01, position=0.5 * d * ax, rotation=q[1])
        cases.append(pair_case(f"c1_like_{k}", a, b, 0.0))
        if k == 0:
            cases.append(pair_case("c1_like_0_exhaustive", a, b, 0.0, exhaustive=True))
    # c2-shaped: domino neighbours
    v, f = S.box((0.1, 0.5, 1.0))
    tilt = rng.uniform(0.0, 0.3, size=12)
    doms = []
    for i in range(12):
        q = np.array([np.cos(0.5 * tilt[i]), 0.0, np.sin(0.5 * tilt[i]), 0.0])
        doms.append(ref_particle(i, v, f, 1e-3, position=(0.18 * i, 0.0, 0.5), rotation=q))
    for i in range(11):
        for j in range(i + 1, min(i + 7, 12)):
            if 0.18 * (j - i) <= 2 * doms[i].sphere.radius:
                cases.append(pair_case(f"c2_like_{i}_{j}", doms[i], doms[j], 0.0))
    # c3-shaped: rock pairs, touching-ish
    for k in range(10):
        va, fa = S.rock(rng)
        vb, fb = S.rock(rng)
        ra, rb = np.exp(rng.uniform(np.log(0.5), np.log(5.0), 2))
        q = S.random_quaternions(rng, 2)
        ax = S.unit_vectors(rng, 1)[0]
        d = (ra + rb) * rng.uniform(0.85, 1.0)
        a = ref_particle(0, va * ra, fa, 0.005, position=-0.5 * d * ax, rotation=q[0])
        b = ref_particle(1, vb * rb, fb, 0.005, position=0.5 * d * ax, rotation=q[1])
        cases.append(pair_case(f"c3_like_{k}", a, b, 0.0))
    # c4-shaped: moving icosphere pairs
    for k, sub in enumerate((1, 1, 2, 2)):
        v0, f = S.icosphere(sub)
        va = v0 * (1 + rng.uniform(-0.05, 0.05, len(v0)))[:, None]
        vb = v0 * (1 + rng.uniform(-0.05, 0.05, len(v0)))[:, None]
        q = S.random_quaternions(rng, 2)
        ax = S.unit_vectors(rng, 1)[0]
        ra = np.linalg.norm(va, axis=1).max() + 1e-3
        rb = np.linalg.norm(vb, axis=1).max() + 1e-3
        gap = rng.uniform(0.0, 0.1)
        vel = rng.normal(0.0, 1.0, (2, 3))
        vel[0] += 1.5 * ax
        vel[1] -= 1.5 * ax
        spin = rng.normal(0.0, 2.0, (2, 3))
        a = ref_particle(0, va, f, 1e-3, position=-0.5 * (ra + rb + gap) * ax, rotation=q[0],
                         velocity=vel[0], angular_velocity=spin[0])
        b = ref_particle(1, vb, f, 1e-3, position=0.5 * (ra + rb + gap) * ax, rotation=q[1],
                         velocity=vel[1], angular_velocity=spin[1])
        cases.append(pair_case(f"c4_like_{k}", a, b, 0.1))
    # c5-shaped: a mixed cluster
    parts = {}
    specs = [(0, "ico", 3, 1.0, (0.0, 0.0, 0.0)), (1, "ico", 0, 0.3, (1.32, 0.0, 0.0)),
             (2, "box", 0, 0.5, (0.0, 1.3, 0.1)), (3, "ico", 2, 0.6, (-1.2, -1.0, 0.3)),
             (4, "ico", 1, 0.1, (0.0, 0.0, 1.12))]
    for pid, kind, sub, r, pos in specs:
        if kind == "ico":
            v, f = S.icosphere(sub)
            v = v * r
        else:
            v, f = S.box((r, 0.8 * r, 0.6 * r))
        vel = rng.normal(0.0, 1.0, 3)
        spin = rng.normal(0.0, 1.0, 3)
        parts[pid] = ref_particle(pid, v, f, 1e-3, position=np.array(pos), velocity=vel,
                                  rotation=S.random_quaternions(rng, 1)[0], angular_velocity=spin)
    floor = make_static(-3, make_plane((-4.0, -4.0, -1.3), (4.0, 4.0, -1.3)), epsilon=1e-3)
    pairs = [(0, 1), (0, 2), (0, 3), (0, 4), (1, 4), (2, 3), (3, -3), (0, -3)]
    cases.append(cluster_case("c5_like_cluster", Cluster(members=(0, 1, 2, 3, 4), t_current=0.25,
                                                         dt=0.1), parts, {-3: floor}, pairs))
    return {"cases": cases}


# ------------------------------------------------------------------ bench-shaped scenes

def _ref_body(raw, pid):
    v, f = raw["meshes"][pid]
    st = raw["states"][pid]
    return ref_particle(pid, v, f, raw["eps"], position=st.position, velocity=st.velocity,
                        rotation=st.rotation, angular_velocity=st.angular_velocity)


def _c4_job(k):
    raw = _BASE["c4"]
    ia, ib = raw["pairs"][k]
    t0 = time.time()
    case = pair_case(f"c4_bench_pair_{k}", _ref_body(raw, ia), _ref_body(raw, ib), raw["dt"], dedup=True)
    case["bench_index"] = int(k)
    case["ref_seconds"] = time.time() - t0
    return case


def _c5_job(p):
    raw = _BASE["c5"]
    sel = np.flatnonzero(raw["problem"] == p)
    pairs = [raw["pairs"][i] for i in sel]
    members = sorted({x for pr in pairs for x in pr})
    parts = {pid: _ref_body(raw, pid) for pid in members}
    t0 = time.time()
    case = cluster_case(f"c5_bench_cluster_{p}", Cluster(members=tuple(members), t_current=0.0, dt=raw["dt"]),
                        parts, {}, pairs, dedup=True)
    case["bench_index"] = int(p)
    case["ref_seconds"] = time.time() - t0
    return case


_BASE = {}


def c4_bench_picks(raw, n_hit=4, n_graze=3, n_other=3):
    """Pairs of the c4 bench workload (BASELINE configs[3], 8192 pairs):
    the ones whose closing speed along the centre line covers the gap by the
    widest margin (hits), the ones it covers by about zero (grazes), and
    seeded random others."""
    dt = raw["dt"]
    n = len(raw["pairs"])
    margin = np.empty(n)
    for k, (ia, ib) in enumerate(raw["pairs"]):
        closing = float(np.dot(raw["states"][ia].velocity - raw["states"][ib].velocity, raw["axes"][k]))
        margin[k] = closing * dt - raw["gaps"][k]
    hits = list(np.argsort(-margin)[:n_hit])
    graze = [int(k) for k in np.argsort(np.abs(margin)) if k not in hits][:n_graze]
    rng = np.random.default_rng(7)
    others = [int(k) for k in rng.permutation(n) if k not in hits and k not in graze][:n_other]
    return [int(k) for k in hits] + graze + others


def c5_bench_picks(raw, big_kind=5, box_kind=6, max_members=6, limit=5):
    """Clusters of the c5 bench workload (BASELINE configs[4]) holding a
    20480-triangle icosphere and a 12-triangle box, smallest first."""
    out = []
    for p in range(raw["n_problems"]):
        sel = np.flatnonzero(raw["problem"] == p)
        members = sorted({x for i in sel for x in raw["pairs"][i]})
        kinds = raw["kinds"][members]
        if (kinds == big_kind).any() and (kinds == box_kind).any() and len(members) <= max_members:
            out.append((len(members), p))
    return [p for _, p in sorted(out)[:limit]]


def c5_impact_picks(raw, big_kind=5, box_kind=6, limit=3):
    """Sphere-box pairs of the c5 bench workload (inside its large clusters)
    whose closing speed covers the bounding-sphere gap within dt by the
    widest margin: each becomes a one-pair cluster (the 20480-triangle tree
    descending against the box's [12, 3, 1] levels, with an impact)."""
    dt = raw["dt"]
    cand = []
    for i, (a, b) in enumerate(raw["pairs"]):
        ka, kb = raw["kinds"][a], raw["kinds"][b]
        if {int(ka), int(kb)} != {big_kind, box_kind}:
            continue
        sa, sb = raw["states"][a], raw["states"][b]
        d = sb.position - sa.position
        dist = float(np.linalg.norm(d))
        gap = dist - raw["radius"][a] - raw["radius"][b]
        closing = float(np.dot(sa.velocity - sb.velocity, d / dist))
        cand.append((closing * dt - gap, i))
    return [i for _, i in sorted(cand, reverse=True)[:limit]]


def _c5_pair_job(i):
    raw = _BASE["c5"]
    a, b = raw["pairs"][i]
    parts = {a: _ref_body(raw, a), b: _ref_body(raw, b)}
    t0 = time.time()
    case = cluster_case(f"c5_bench_pair_{i}", Cluster(members=(a, b), t_current=0.0, dt=raw["dt"]),
                        parts, {}, [(a, b)], dedup=True)
    case["bench_pair"] = int(i)
    case["ref_seconds"] = time.time() - t0
    return case


def gen_scenes_baseline(workers=8):
    """c4 pairs and c5 clusters taken from the bench workloads themselves
    (scenes.config4_raw / config5_raw at their BASELINE sizes), rebuilt with
    the reference's make_particle and run through the reference."""
    import multiprocessing as mp

    _BASE["c4"] = S.config4_raw()
    _BASE["c5"] = S.config5_raw()
    c4 = c4_bench_picks(_BASE["c4"])
    c5 = c5_bench_picks(_BASE["c5"])
    c5p = c5_impact_picks(_BASE["c5"])
    print("c4 pairs", c4, "c5 clusters", c5, "c5 impact pairs", c5p, flush=True)
    with mp.get_context("fork").Pool(workers) as pool:
        r5 = pool.map_async(_c5_job, c5, chunksize=1)
        r5p = pool.map_async(_c5_pair_job, c5p, chunksize=1)
        r4 = pool.map_async(_c4_job, c4, chunksize=1)
        cases = r4.get() + r5.get() + r5p.get()
    for c in cases:
        print(c["name"], "collision", c["result"]["collision"], "raw", len(c["result"]["raw"]["t"]),
              "rows", c["rows"], f"{c['ref_seconds']:.1f}s", flush=True)
    return {"cases": cases}


# ------------------------------------------------------------------ engine sweeps

def gen_engine_sweeps(n_sweeps=30):
    """The reference engine (`ltsdem.engine.step`, engine.py:146-261) on its
    own "stacks" scenario (one row of boxes on a floor: clusters fall out of
    step, so held-back clusters are reused from the engine's cache).  Per
    sweep: every cluster with its cache-key fields, its result and whether
    the engine computed it (cache miss) -- recorded by wrapping the module
    globals `compute_effective_dt` and `mask_clusters` that step() resolves
    at call time -- plus the particle states the narrow phase saw.
    tests/test_gpu_sweep.py replays the sweeps through
    paper_2309_15417_b200.sweep.SweepDriver."""
    from ltsdem import engine
    from ltsdem.scenarios import ScenarioConfig, build_world

    world = build_world(ScenarioConfig("stacks", rows=1, seed=3))
    calls = {}
    sweeps = []
    bodies0 = []
    f_ced, f_mask = engine.compute_effective_dt, engine.mask_clusters

    def ced(cluster, particles, statics, pairs, **kw):
        res = f_ced(cluster, particles, statics, pairs, **kw)
        calls[tuple(cluster.members)] = [tuple(p) for p in pairs]
        return res

    def soa(rows, n3=False):
        return np.array(rows, dtype=np.float64).reshape(-1, 3) if n3 else np.array(rows)

    def mask(clusters, results):
        parts = world.particles
        ids = sorted(parts)
        cur = [parts[pid].timeline.current for pid in ids]
        rec = {"ids": np.array(ids, dtype=np.int64),
               "position": np.array([c.position for c in cur]), "velocity": np.array([c.velocity for c in cur]),
               "rotation": np.array([c.rotation for c in cur]),
               "angular_velocity": np.array([c.angular_velocity for c in cur]),
               "t": np.array([c.t for c in cur]),
               "version": np.array([parts[pid].timeline.version for pid in ids], dtype=np.int64)}
        if not sweeps:
            bodies0[:] = [SC.encode_body(parts[pid]) for pid in ids]
        mem, moff, sta, soff, prs, poff, cts, coff = [], [0], [], [0], [], [0], [], [0]
        for c, r in zip(clusters, results):
            m = tuple(c.members)
            mem += list(m)
            moff.append(len(mem))
            sta += list(c.statics)
            soff.append(len(sta))
            prs += calls.get(m, [])
            poff.append(len(prs))
            cts += list(r.contacts)
            coff.append(len(cts))
        rec.update({
            "members": np.array(mem, dtype=np.int64), "members_off": np.array(moff, dtype=np.int64),
            "statics": np.array(sta, dtype=np.int64), "statics_off": np.array(soff, dtype=np.int64),
            "t_current": np.array([c.t_current for c in clusters]), "dt": np.array([c.dt for c in clusters]),
            "computed": np.array([tuple(c.members) in calls for c in clusters]),
            "pairs": np.array(prs, dtype=np.int64).reshape(-1, 2), "pairs_off": np.array(poff, dtype=np.int64),
            "res_dt": np.array([r.dt for r in results]),
            "res_collision": np.array([r.collision for r in results]),
            "res_first": np.array([np.nan if r.first_contact is None else r.first_contact for r in results]),
            "res_narrowing": np.array([r.narrowing_iters for r in results], dtype=np.int64),
            "contacts": SC.encode_contacts(cts), "contacts_off": np.array(coff, dtype=np.int64)})
        sweeps.append(rec)
        calls.clear()
        return f_mask(clusters, results)

    engine.compute_effective_dt, engine.mask_clusters = ced, mask
    try:
        for _ in range(n_sweeps):
            engine.step(world)
    finally:
        engine.compute_effective_dt, engine.mask_clusters = f_ced, f_mask
    statics = [SC.encode_body(s) for s in world.statics.values()]
    n_comp = sum(int(sw["computed"].sum()) for sw in sweeps)
    n_all = sum(len(sw["dt"]) for sw in sweeps)
    n_coll = sum(int(sw["res_collision"].sum()) for sw in sweeps)
    n_spin = sum(int(np.any(sw["angular_velocity"] != 0.0)) for sw in sweeps)
    print(f"engine sweeps: {len(sweeps)} sweeps, {n_all} clusters, {n_comp} computed, {n_coll} colliding, "
          f"{n_spin} sweeps with spinning particles", flush=True)
    return {"sweeps": sweeps, "statics": statics, "bodies": bodies0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    rng = np.random.default_rng(20251020)
    jobs = {
        "kernels": lambda: gen_kernels(np.random.default_rng(101)),
        "witness": lambda: gen_witness(np.random.default_rng(102)),
        "fusion": lambda: gen_fusion(np.random.default_rng(103)),
        "trees": lambda: gen_trees(np.random.default_rng(104)),
        "scenes_ccd": gen_scenes_ccd,
        "scenes_configs": lambda: gen_scenes_configs(np.random.default_rng(105)),
        "scenes_crit2": lambda: gen_scenes_crit2(limit=40 if args.quick else 200),
        "scenes_baseline": gen_scenes_baseline,
        "engine_sweeps": gen_engine_sweeps,
    }
    del rng
    for name, job in jobs.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        data = job()
        gio.save(os.path.join(HERE, f"{name}.npz"), data)
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
