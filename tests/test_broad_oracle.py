"""The broad-phase CPU oracle against the reference's own outputs, and the
host side of the broad-phase boundary (packing, graph assembly), on CPU.

tests/golden/broadphase.npz was produced by running the reference's
`ltsdem.broadphase.build_collision_graph` (broadphase.py:198-252) and
`_min_distance_over_window` (:128-151) on seeded scenes
(tests/golden/make_golden_broad.py).  The oracle must reproduce the graphs
bit for bit -- edge order, windows, links, step bounds -- and the Check-2
distances of the trajectory rows.
"""

import numpy as np
import pytest

from helpers import golden
from oracle import broad_oracle as BO


def _scenes():
    return golden("broadphase")["scenes"]


def graph_of_case(g):
    """The golden graph as (edges dict, links dict, dts)."""
    edges = {(int(a), int(b)): (float(w[0]), float(w[1])) for (a, b), w in zip(g["edges"], g["windows"])}
    links = {}
    for k, p in enumerate(g["link_keys"]):
        links[int(p)] = tuple(int(s) for s in g["link_sids"][g["link_ptr"][k]:g["link_ptr"][k + 1]])
    return edges, links, g["dts"]


@pytest.mark.parametrize("name", [g["name"] for g in golden("broadphase")["scenes"]])
def test_oracle_graph_bit_exact(name):
    g = next(s for s in _scenes() if s["name"] == name)
    out = BO.build_collision_graph(g["rec"], g["srec"], g["pids"], g["sids"], g["dt_max"], g["growth"])
    edges, links, dts = graph_of_case(g)
    np.testing.assert_array_equal(np.array([out.dts[int(p)] for p in g["pids"]]), dts)
    assert list(out.edges.items()) == list(edges.items())  # same order, same windows (bit for bit)
    assert list(out.static_links.items()) == list(links.items())


def test_oracle_tube_rows_bit_exact():
    r = golden("broadphase")["rows"]
    dist, hit = BO.tube_rows(r["t1"], r["c1"], r["r1"], r["t2"], r["c2"], r["r2"],
                             r["window"][:, 0], r["window"][:, 1])
    np.testing.assert_array_equal(dist, r["dist"])
    np.testing.assert_array_equal(hit, r["hit"])
    assert r["hit"].sum() > 30 and (~r["hit"]).sum() > 30  # both verdicts exercised


def test_fixtures_cover_the_reference_cases():
    names = {g["name"] for g in _scenes()}
    assert {"approaching", "receding", "timing_screen", "static_link", "far_static", "two_statics"} <= names
    big = [g for g in _scenes() if len(g["pids"]) >= 2000]
    assert big and all(len(g["edges"]) > 100 for g in big)
    assert any(len(g["link_sids"]) > 100 for g in _scenes())


def test_packing_matches_the_fixture_layout():
    """The product's packer reads the reference's fields into the record
    layout include/ltsgpu.h documents (the fixture's records were packed by
    the generator's own code)."""
    from paper_2309_15417_b200 import bodies as B
    from paper_2309_15417_b200 import broadphase as BP

    rng = np.random.default_rng(3)
    parts = {}
    for pid in (5, 1, 3):
        st = B.state(rng.normal(size=3), velocity=rng.normal(size=3), rotation=(0.5, 0.5, 0.5, 0.5),
                     angular_velocity=rng.normal(size=3), t=0.25)
        p = B.Particle(pid=pid, tree=None, epsilon=0.01, radius=0.7, timeline=B.timeline(st))
        p.timeline.old.t = 0.125
        parts[pid] = p
    rec = BP.pack_particles(parts)
    assert rec.shape == (3, BP.RECORD)
    p = parts[1]
    np.testing.assert_array_equal(rec[0, 8:11], p.timeline.current.position)
    assert rec[0, 7] == 0.125 and rec[0, 15] == 0.25 and rec[0, 25] == 0.7
    np.testing.assert_array_equal(rec[0, 22:25], 0.0)
    stat = B.StaticBody(sid=-2, tree=None, epsilon=0.01, sphere=B.BoundingSphere(np.ones(3), 2.0))
    np.testing.assert_array_equal(BP.pack_statics({-2: stat}), [[1.0, 1.0, 1.0, 2.0]])


def test_host_policy_helpers_match_the_reference():
    from paper_2309_15417_b200 import broadphase as BP

    assert BP.pair_window(1.0, 0.5, 0.8, 0.3) == (0.8, 0.8 + 0.3)
    with pytest.raises(ValueError):
        BP.TimeStepPolicy(dt_max=0.0)
    with pytest.raises(ValueError):
        BP.TimeStepPolicy(dt_max=1.0, growth=1.0)
    from types import SimpleNamespace as NS

    tl = NS(old=NS(t=0.0), current=NS(t=0.1))
    assert BP.particle_dt(tl, BP.TimeStepPolicy(dt_max=1.0)) == 2.0 * 0.1
    assert BP.particle_dt(NS(old=NS(t=0.3), current=NS(t=0.3)), BP.TimeStepPolicy(dt_max=0.25)) == 0.25


def test_static_sphere_restatement_matches_the_reference_fixture():
    """bodies.bounding_sphere restates mesh.bounding_sphere (mesh.py:335-352):
    the fixture's static spheres were built by the reference's make_static."""
    from paper_2309_15417_b200 import bodies as B

    g = next(s for s in _scenes() if s["name"] == "static_link")
    v = np.array([[-5.0, -5.0, 0.0], [5.0, -5.0, 0.0], [5.0, 5.0, 0.0], [-5.0, 5.0, 0.0]])
    sph = B.bounding_sphere(v, 0.01)
    np.testing.assert_array_equal(np.r_[sph.center, sph.radius], g["srec"][0])
