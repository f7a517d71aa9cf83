"""Generate the broad-phase golden fixtures by running the REFERENCE itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_broad.py

Output (committed): tests/golden/broadphase.npz with

* `scenes`: collision graphs of `ltsdem.broadphase.build_collision_graph`
  (broadphase.py:198-252) on seeded scenes -- the reference's own
  test_broadphase.py scenes and its `_random_scene` generator
  (tests/test_broadphase.py:20-37, :124-137), a dense 400-cube scene with
  floor and walls, off-centre spinning spheres, and the c5 workload's 2000
  particles (fresh and with step histories).  Each scene stores the packed
  inputs (the record layout of include/ltsgpu.h) and the graph: edges in
  dict order with their windows, static links in dict order, step bounds.
* `rows`: Check 2 on explicit trajectory pairs drawn by the reference's
  `_random_trajectory_pair` (test_broadphase.py:155-169): the minimum
  centre distance `_min_distance_over_window` (:128-151) and the verdict.
"""

from __future__ import annotations

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

from ltsdem import broadphase as RB  # noqa: E402
from ltsdem.body import Particle, initial_state, make_static  # noqa: E402
from ltsdem.mesh import BoundingSphere, make_plane  # noqa: E402
from ltsdem.state import make_timeline  # noqa: E402

import gio  # noqa: E402
import test_broadphase as RT  # noqa: E402  (the reference's own test helpers)
from paper_2309_15417_b200 import scenes as S  # noqa: E402


def pack(particles, statics):
    pids, sids = sorted(particles), sorted(statics)
    rec = np.zeros((len(pids), 28))
    for k, pid in enumerate(pids):
        p = particles[pid]
        o, c = p.timeline.old, p.timeline.current
        rec[k, 0:3], rec[k, 3:7], rec[k, 7] = o.position, o.rotation, o.t
        rec[k, 8:11], rec[k, 11:15], rec[k, 15] = c.position, c.rotation, c.t
        rec[k, 16:19], rec[k, 19:22] = c.velocity, c.angular_velocity
        rec[k, 22:25], rec[k, 25] = p.sphere.center, p.sphere.radius
    srec = np.zeros((len(sids), 4))
    for k, sid in enumerate(sids):
        srec[k, 0:3], srec[k, 3] = statics[sid].sphere.center, statics[sid].sphere.radius
    return rec, srec, np.array(pids, dtype=np.int64), np.array(sids, dtype=np.int64)


def record(name, particles, statics, policy, tol=False):
    t0 = time.perf_counter()
    g = RB.build_collision_graph(particles, statics, policy)
    wall = time.perf_counter() - t0
    rec, srec, pids, sids = pack(particles, statics)
    edges = np.array(list(g.edges.keys()), dtype=np.int64).reshape(-1, 2)
    windows = np.array(list(g.edges.values()), dtype=np.float64).reshape(-1, 2)
    link_keys = np.array(list(g.static_links.keys()), dtype=np.int64)
    link_ptr = np.concatenate([[0], np.cumsum([len(v) for v in g.static_links.values()])]).astype(np.int64)
    link_sids = np.array([s for v in g.static_links.values() for s in v], dtype=np.int64)
    dts = np.array([g.dts[p] for p in pids], dtype=np.float64)
    print(f"  {name}: {len(pids)} particles, {len(sids)} statics, {len(edges)} edges, "
          f"{len(link_sids)} links, reference {wall:.2f} s", flush=True)
    return {"name": name, "rec": rec, "srec": srec, "pids": pids, "sids": sids,
            "dt_max": float(policy.dt_max), "growth": float(policy.growth), "edges": edges,
            "windows": windows, "link_keys": link_keys, "link_ptr": link_ptr, "link_sids": link_sids,
            "dts": dts, "sincos": bool(tol), "ref_wall_s": wall}


def sphere_particle(pid, radius, state, centre=(0.0, 0.0, 0.0), eps=1e-3):
    """A Particle whose broad-phase inputs (timeline, sphere) are set directly;
    the broad phase reads nothing else (broadphase.py:83-95)."""
    return Particle(pid=pid, mesh=None, tree=None, epsilon=eps, mass=None,
                    sphere=BoundingSphere(center=np.asarray(centre, dtype=float), radius=float(radius)),
                    timeline=make_timeline(state))


def ref_test_scenes():
    out = []
    a = RT._cube_particle(0, (-2.0, 0.0, 0.0), velocity=(1.0, 0.0, 0.0))
    b = RT._cube_particle(1, (2.0, 0.0, 0.0), velocity=(-1.0, 0.0, 0.0))
    out.append(record("approaching", {0: a, 1: b}, {}, RB.TimeStepPolicy(dt_max=5.0)))
    a = RT._cube_particle(0, (-2.0, 0.0, 0.0), velocity=(-1.0, 0.0, 0.0))
    b = RT._cube_particle(1, (2.0, 0.0, 0.0), velocity=(1.0, 0.0, 0.0))
    out.append(record("receding", {0: a, 1: b}, {}, RB.TimeStepPolicy(dt_max=5.0)))
    a = RT._cube_particle(0, (10.0, 0.0, 0.0), velocity=(-3.0, 0.0, 0.0))
    RT._advance(a, 1.0)
    b = RT._cube_particle(1, (0.0, 0.0, 0.0))
    out.append(record("timing_screen", {0: a, 1: b}, {}, RB.TimeStepPolicy(dt_max=4.0)))
    floor = make_static(-1, make_plane((-5.0, -5.0, 0.0), (5.0, 5.0, 0.0)), epsilon=0.01)
    p = RT._cube_particle(0, (0.0, 0.0, 2.0), velocity=(0.0, 0.0, -1.0))
    out.append(record("static_link", {0: p}, {-1: floor}, RB.TimeStepPolicy(dt_max=4.0)))
    p = RT._cube_particle(0, (0.0, 0.0, 50.0), velocity=(0.0, 0.0, 1.0))
    out.append(record("far_static", {0: p}, {-1: floor}, RB.TimeStepPolicy(dt_max=1.0)))
    s1 = make_static(-1, make_plane((-1.0, -1.0, 0.0), (1.0, 1.0, 0.0)), epsilon=0.01)
    s2 = make_static(-2, make_plane((-1.0, -1.0, 0.1), (1.0, 1.0, 0.1)), epsilon=0.01)
    p = RT._cube_particle(0, (30.0, 0.0, 0.0))
    out.append(record("two_statics", {0: p}, {-1: s1, -2: s2}, RB.TimeStepPolicy(dt_max=0.5)))
    return out


def random_scenes():
    out = []
    for seed in range(6):
        rng = np.random.default_rng(seed)
        particles, statics = RT._random_scene(rng, 24)
        out.append(record(f"random_{seed}", particles, statics, RB.TimeStepPolicy(dt_max=0.6)))
    return out


def dense_scene(n=400, seed=21):
    rng = np.random.default_rng(seed)
    particles = {}
    for pid in range(n):
        p = RT._cube_particle(pid, rng.uniform(0.0, 12.0, size=3), velocity=rng.normal(scale=2.0, size=3),
                              omega=rng.normal(scale=1.0, size=3), t=float(rng.choice([0.0, 0.25])))
        if rng.uniform() < 0.6:
            RT._advance(p, float(rng.uniform(0.02, 0.5)), new_velocity=rng.normal(scale=2.0, size=3))
        particles[pid] = p
    statics = {
        -1: make_static(-1, make_plane((-30.0, -30.0, -1.0), (30.0, 30.0, -1.0)), 0.01),
        -2: make_static(-2, make_plane((-1.5, 0.0, 0.0), (-1.5, 14.0, 14.0)), 0.01),
        -3: make_static(-3, make_plane((0.0, 13.0, 0.0), (14.0, 13.0, 14.0)), 0.01),
    }
    return [record("dense_400", particles, statics, RB.TimeStepPolicy(dt_max=0.4, growth=1.5))]


def offcentre_scene(n=120, seed=33):
    rng = np.random.default_rng(seed)
    particles = {}
    for pid in range(n):
        st = initial_state(rng.uniform(0.0, 6.0, size=3), velocity=rng.normal(scale=1.0, size=3),
                           rotation=S.random_quaternions(rng, 1)[0],
                           angular_velocity=rng.normal(scale=3.0, size=3))
        particles[pid] = sphere_particle(pid, rng.uniform(0.2, 0.6), st, centre=rng.normal(scale=0.3, size=3))
    return [record("offcentre_spin", particles, {}, RB.TimeStepPolicy(dt_max=0.3), tol=True)]


def c5_scenes():
    raw = S.config5_raw()
    out = []
    for hist in (False, True):
        rng = np.random.default_rng(55)
        particles = {}
        for i, (st, r) in enumerate(zip(raw["states"], raw["radius"])):
            p = sphere_particle(i, r, initial_state(st.position, velocity=st.velocity, rotation=st.rotation,
                                                    angular_velocity=st.angular_velocity))
            if hist and rng.uniform() < 0.5:
                RT._advance(p, float(rng.uniform(0.01, 0.08)), new_velocity=rng.normal(scale=1.0, size=3))
            particles[i] = p
        out.append(record("c5_history" if hist else "c5_fresh", particles, {},
                          RB.TimeStepPolicy(dt_max=raw["dt"])))
    return out


def trajectory_rows(n=600, seed=11):
    rng = np.random.default_rng(seed)
    t1, c1, r1, t2, c2, r2, win, dist, hit = ([] for _ in range(9))
    for _ in range(n):
        ta, tb, window = RT._random_trajectory_pair(rng)
        t1.append(ta.times), c1.append(ta.centers), r1.append(ta.radius)
        t2.append(tb.times), c2.append(tb.centers), r2.append(tb.radius)
        win.append(window)
        dist.append(RB._min_distance_over_window(ta, tb, window))
        hit.append(RB.check_spacetime_tube(ta, tb, window))
    # the reference's empty-window case (test_broadphase.py:203-208) and a
    # zero-length window (a single knot)
    a = RT._cube_particle(0, (0.0, 0.0, 0.0))
    b = RT._cube_particle(1, (0.5, 0.0, 0.0))
    ta, tb = RB._Trajectory.of_particle(a, 0.1), RB._Trajectory.of_particle(b, 0.1)
    for window in ((1.0, 0.5), (0.05, 0.05)):
        t1.append(ta.times), c1.append(ta.centers), r1.append(ta.radius)
        t2.append(tb.times), c2.append(tb.centers), r2.append(tb.radius)
        win.append(window)
        dist.append(RB._min_distance_over_window(ta, tb, window))
        hit.append(RB.check_spacetime_tube(ta, tb, window))
    return {"t1": np.array(t1), "c1": np.array(c1), "r1": np.array(r1), "t2": np.array(t2),
            "c2": np.array(c2), "r2": np.array(r2), "window": np.array(win), "dist": np.array(dist),
            "hit": np.array(hit)}


def main():
    print("broad-phase goldens (reference run)", flush=True)
    scenes = ref_test_scenes() + random_scenes() + dense_scene() + offcentre_scene() + c5_scenes()
    rows = trajectory_rows()
    gio.save(os.path.join(HERE, "broadphase.npz"), {"scenes": scenes, "rows": rows})
    print("wrote broadphase.npz")


if __name__ == "__main__":
    main()
