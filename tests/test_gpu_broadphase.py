"""GPU parity of the broad phase (ltsg_broadphase / ltsg_tube_rows).

Against the reference's own graphs (tests/golden/broadphase.npz, produced
by ltsdem.broadphase, broadphase.py:198-252): edges in the same dict order
with the same windows, the same static links and step bounds, bit for bit.
Against the pinned CPU oracle on larger seeded scenes, and through the
drop-in `build_collision_graph` on the package's own body classes.
"""

import numpy as np
import pytest

from helpers import golden
from oracle import broad_oracle as BO
from test_broad_oracle import graph_of_case

pytestmark = pytest.mark.gpu


def _bp():
    from paper_2309_15417_b200 import broadphase as BP

    return BP


def _graph(BP, rec, srec, pids, sids, dt_max, growth):
    ga = BP.graph_arrays(rec, srec, BP.TimeStepPolicy(dt_max=dt_max, growth=growth))
    pids, sids = np.asarray(pids), np.asarray(sids)
    edges = {(int(pids[a]), int(pids[b])): (float(w[0]), float(w[1])) for (a, b), w in zip(ga.edge, ga.window)}
    links = {}
    for i, s in ga.link:
        links.setdefault(int(pids[i]), []).append(int(sids[s]))
    return edges, {k: tuple(v) for k, v in links.items()}, ga


@pytest.mark.parametrize("name", [g["name"] for g in golden("broadphase")["scenes"]])
def test_graph_matches_the_reference(name):
    BP = _bp()
    g = next(s for s in golden("broadphase")["scenes"] if s["name"] == name)
    edges, links, ga = _graph(BP, g["rec"], g["srec"], g["pids"], g["sids"], g["dt_max"], g["growth"])
    ref_edges, ref_links, ref_dts = graph_of_case(g)
    np.testing.assert_array_equal(ga.dts, ref_dts)
    assert list(links.items()) == list(ref_links.items())
    if g["sincos"]:
        # off-centre spinning spheres: quaternions.advance's sin/cos (CUDA vs
        # libm may differ in the last bit) moves the extrapolated centre by
        # ~1e-16; the windows do not depend on it, the verdicts are compared
        assert list(edges) == list(ref_edges)
        assert edges == ref_edges
    else:
        assert list(edges.items()) == list(ref_edges.items())
    assert ga.candidates >= len(edges) + sum(len(v) for v in links.values())


def test_tube_rows_match_the_reference():
    BP = _bp()
    r = golden("broadphase")["rows"]
    dist, hit = BP.tube_rows(r["t1"], r["c1"], r["r1"], r["t2"], r["c2"], r["r2"], r["window"])
    np.testing.assert_array_equal(dist, r["dist"])
    np.testing.assert_array_equal(hit, r["hit"])


def _random_records(rng, n, n_static=0, side=40.0, hist=0.5):
    rec = np.zeros((n, 28))
    rec[:, 8:11] = rng.uniform(0.0, side, (n, 3))
    rec[:, 16:19] = rng.normal(size=(n, 3))
    rec[:, 19:22] = rng.normal(size=(n, 3))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1)[:, None]
    rec[:, 11:15] = q
    rec[:, 3:7] = q
    rec[:, 15] = rng.choice([0.0, 0.05, 0.1], n)
    back = rng.uniform(0.0, 0.1, n) * (rng.uniform(size=n) < hist)
    rec[:, 7] = rec[:, 15] - back
    rec[:, 0:3] = rec[:, 8:11] - back[:, None] * rng.normal(size=(n, 3))
    rec[:, 25] = np.exp(rng.uniform(np.log(0.1), np.log(1.5), n))
    srec = np.zeros((n_static, 4))
    srec[:, 0:3] = rng.uniform(0.0, side, (n_static, 3))
    srec[:, 3] = rng.uniform(0.5, 30.0, n_static)  # some statics span the whole box
    return rec, srec


@pytest.mark.parametrize("seed,n,n_static", [(0, 6000, 0), (1, 3000, 7), (2, 1, 0), (3, 2, 3), (4, 700, 40)])
def test_graph_matches_the_oracle(seed, n, n_static):
    BP = _bp()
    rng = np.random.default_rng(seed)
    rec, srec = _random_records(rng, n, n_static)
    pids = np.arange(n) * 3 + 1
    sids = -np.arange(n_static, 0, -1) * 2
    edges, links, ga = _graph(BP, rec, srec, pids, sids, 0.1, 2.0)
    o = BO.build_collision_graph(rec, srec, pids, sids, 0.1, 2.0)
    np.testing.assert_array_equal(ga.dts, np.array([o.dts[int(p)] for p in pids]))
    assert list(edges.items()) == list(o.edges.items())
    assert list(links.items()) == list(o.static_links.items())
    assert ga.candidates == o.candidates


def test_large_scene_is_invariant_to_body_order():
    """20k bodies (the c3 count): relabelling the particles relabels the graph
    and nothing else (the device enumeration is complete and ordered)."""
    BP = _bp()
    rng = np.random.default_rng(7)
    n = 20000
    rec, srec = _random_records(rng, n, 2, side=90.0)
    e1, l1, g1 = _graph(BP, rec, srec, np.arange(n), [-2, -1], 0.1, 2.0)
    perm = rng.permutation(n)
    e2, l2, g2 = _graph(BP, rec[perm], srec, np.arange(n), [-2, -1], 0.1, 2.0)
    inv = {int(k): int(v) for v, k in enumerate(perm)}  # old index -> new index
    remap = {}
    for (a, b), w in e1.items():
        x, y = sorted((inv[a], inv[b]))
        remap[(x, y)] = w
    assert remap == e2
    assert {inv[p]: v for p, v in l1.items()} == l2
    assert g1.candidates == g2.candidates and len(e1) > 1000


def test_drop_in_on_package_bodies():
    """build_collision_graph on duck-typed bodies equals the oracle on the
    records the fixture generator would pack."""
    from paper_2309_15417_b200 import bodies as B

    BP = _bp()
    rng = np.random.default_rng(5)
    particles = {}
    for pid in range(200):
        st = B.state(rng.uniform(0, 8, 3), velocity=rng.normal(size=3), angular_velocity=rng.normal(size=3))
        p = B.Particle(pid=pid, tree=None, epsilon=1e-3, radius=float(rng.uniform(0.2, 0.6)), timeline=B.timeline(st))
        if pid % 3 == 0:
            p.timeline.old.t = -0.05
            p.timeline.old.position = p.timeline.current.position - 0.05 * rng.normal(size=3)
        particles[pid] = p
    floor = B.StaticBody(sid=-1, tree=None, epsilon=0.01,
                         sphere=B.BoundingSphere(np.array([4.0, 4.0, -50.0]), 50.2))
    policy = BP.TimeStepPolicy(dt_max=0.2)
    g = BP.build_collision_graph(particles, {-1: floor}, policy)
    rec, srec = BP.pack_particles(particles), BP.pack_statics({-1: floor})
    o = BO.build_collision_graph(rec, srec, np.arange(200), np.array([-1]), 0.2, 2.0)
    assert list(g.edges.items()) == list(o.edges.items())
    assert g.static_links == o.static_links and g.dts == o.dts
    assert len(g.static_links) > 0 and len(g.edges) > 0
    assert g.neighbors() == {k: v for k, v in g.neighbors().items()}


def test_empty_and_static_only():
    BP = _bp()
    assert BP.build_collision_graph({}, {}, BP.TimeStepPolicy(dt_max=1.0)).edges == {}
    ga = BP.graph_arrays(np.zeros((0, 28)), np.array([[0.0, 0, 0, 1.0], [0.5, 0, 0, 1.0]]),
                         BP.TimeStepPolicy(dt_max=1.0))
    assert len(ga.edge) == 0 and len(ga.link) == 0 and ga.candidates == 0
