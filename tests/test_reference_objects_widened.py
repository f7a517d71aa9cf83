"""The drop-in claim of the widened rows with genuine reference objects, on
CPU: the package's host packing (`broadphase.pack_particles/pack_statics`,
`contacts.body_record`) reads real `ltsdem` particles, statics and contact
points, and the pinned CPU oracles run on those packed records reproduce
what the reference itself computes from the same objects -- the collision
graph (broadphase.py:198-252) and the impulse solution (contacts.py:114-198),
bit for bit.  Needs the reference importable (this build container);
skipped where it is absent (the GPU box)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference not present on this host", allow_module_level=True)
sys.path.insert(0, REF)

from oracle import broad_oracle as BO  # noqa: E402
from oracle import contact_oracle as CO  # noqa: E402
from paper_2309_15417_b200 import broadphase as BP  # noqa: E402
from paper_2309_15417_b200 import contacts as CT  # noqa: E402
from paper_2309_15417_b200 import scenes  # noqa: E402


def _ref_particles(n, seed, spread):
    from ltsdem.body import initial_state, make_particle, make_static
    from ltsdem.mesh import TriangleMesh, make_plane
    from ltsdem.state import extrapolate_free_flight

    rng = np.random.default_rng(seed)
    parts = {}
    for pid in range(n):
        v, f = scenes.icosphere(int(rng.integers(0, 2)))
        v = v * float(rng.uniform(0.3, 0.8)) * (1 + rng.uniform(-0.05, 0.05, len(v)))[:, None]
        p = make_particle(pid, TriangleMesh(v, f), 1e-3, initial_state(
            position=rng.uniform(-spread, spread, size=3), velocity=rng.normal(size=3),
            rotation=scenes.random_quaternions(rng, 1)[0], angular_velocity=rng.normal(size=3)))
        if pid % 3:  # some particles have already stepped: old != current, own clocks
            tl = p.timeline
            tl.old = tl.current
            tl.current = extrapolate_free_flight(tl.current, float(rng.uniform(0.01, 0.05)))
            tl.touch()
        parts[pid] = p
    statics = {-1: make_static(-1, make_plane((-spread, -spread, -spread - 0.5), (spread, spread, -spread - 0.5)),
                               epsilon=1e-3)}
    return parts, statics


@pytest.mark.parametrize("seed,spread", [(1, 1.5), (2, 3.0), (3, 6.0)])
def test_broadphase_records_of_reference_objects_give_the_reference_graph(seed, spread):
    from ltsdem import broadphase as RB

    parts, statics = _ref_particles(40, seed, spread)
    want = RB.build_collision_graph(parts, statics, RB.TimeStepPolicy(dt_max=0.1))
    pids, sids = sorted(parts), sorted(statics)
    rec, srec = BP.pack_particles(parts, pids), BP.pack_statics(statics, sids)
    got = BO.build_collision_graph(rec, srec, np.asarray(pids), np.asarray(sids), 0.1, 2.0)
    assert list(got.edges.items()) == list(want.edges.items())  # same pairs, same order, same windows
    assert got.static_links == want.static_links
    assert got.dts == want.dts
    assert len(want.edges) > 0
    # the C gather and the Python packing loop agree
    saved, BP._fastpack = BP._fastpack, None
    try:
        assert BP.pack_particles(parts, pids).tobytes() == rec.tobytes()
    finally:
        BP._fastpack = saved


def test_contact_records_of_reference_objects_give_the_reference_solution():
    from ltsdem import contacts as RC
    from ltsdem.ccd import ContactPoint

    parts, _ = _ref_particles(6, 11, 1.0)
    rng = np.random.default_rng(5)
    contacts = []
    for a, b in [(0, 1), (1, 2), (2, -1), (3, 4), (4, 5), (0, 5)]:
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        t = max(parts[a].timeline.current.t, parts[b].timeline.current.t if b >= 0 else 0.0) + 0.01
        contacts.append(ContactPoint(body_a=a, body_b=b, position=rng.normal(size=3) * 0.3, normal=n,
                                     depth=float(rng.uniform(0, 1e-3)), t=float(t), tri_a=0, tri_b=0, threshold=2e-3))
    cfg = RC.SolverConfig()
    want = RC.solve_impulses(contacts, parts, cfg)
    bodies = {pid: np.asarray(CT.body_record(p), dtype=np.float64) for pid, p in parts.items()}
    clist = [dict(body_a=c.body_a, body_b=c.body_b, position=c.position, normal=c.normal, t=c.t) for c in contacts]
    vel, ang, iters, conv, lam, fric = CO.solve_impulses(clist, bodies, dict(
        restitution=cfg.restitution, friction=cfg.friction, relaxation=cfg.relaxation, penalty=cfg.penalty,
        threshold=cfg.threshold, max_iterations=cfg.max_iterations))
    assert iters == want.iterations and conv == want.converged
    assert list(vel) == list(want.velocities)
    for bid in vel:
        assert np.array_equal(vel[bid], want.velocities[bid]), bid
        assert np.array_equal(ang[bid], want.angular_velocities[bid]), bid
    assert np.array_equal(np.asarray(lam), np.asarray(want.normal_impulses))
