"""The broad-phase and contact oracles against whole sweeps of the reference
engine (tests/golden/engine_steps.npz, recorded from `ltsdem.engine.step`
by tests/golden/make_golden_engine.py): the collision graph of every sweep,
every `solve_impulses` call and every commit, bit for bit, from records the
package's host packing builds out of the particles' timelines."""

from types import SimpleNamespace as NS

import numpy as np
import pytest

from golden import scene_codec as SC
from helpers import golden
from oracle import broad_oracle as BO
from oracle import contact_oracle as CO
from paper_2309_15417_b200 import bodies as B
from paper_2309_15417_b200 import broadphase as BP
from paper_2309_15417_b200 import contacts as CT


@pytest.fixture(scope="module")
def W():
    G = golden("engine_steps")
    ids = [int(i) for i in G["ids"]]
    parts = {}
    for k, rec in enumerate(G["bodies"]):
        p = SC.decode_body(rec)
        p.mass = NS(mass=1.0 / float(G["mass"]["inv_mass"][k]), inverse_inertia=G["mass"]["inv_inertia"][k].copy())
        p.radius = float(G["spheres"]["radius"][k])
        parts[p.pid] = p
    statics = {}
    for k, rec in enumerate(G["statics"]):
        s = SC.decode_body(rec)
        s.sphere = B.BoundingSphere(center=G["spheres"]["static_center"][k].copy(),
                                    radius=float(G["spheres"]["static_radius"][k]))
        statics[s.sid] = s
    return NS(G=G, ids=ids, parts=parts, statics=statics)


def _set(W, sw):
    for j, pid in enumerate(W.ids):
        tl = W.parts[pid].timeline
        for which in ("old", "current"):
            s = sw[which]
            setattr(tl, which, B.state(s["position"][j], s["velocity"][j], s["rotation"][j],
                                       s["angular_velocity"][j], s["t"][j]))


def _clist(c):
    return [dict(body_a=int(c["body_a"][i]), body_b=int(c["body_b"][i]), position=c["position"][i],
                 normal=c["normal"][i], t=float(c["t"][i]), depth=float(c["depth"][i])) for i in range(len(c["t"]))]


def test_oracles_reproduce_the_engine_run(W):
    G = W.G
    cfg = {k: float(v) for k, v in G["solver"].items()}
    sids = sorted(W.statics)
    n_edges = n_solves = n_commits = 0
    for k, sw in enumerate(G["sweeps"]):
        _set(W, sw)
        rec, srec = BP.pack_particles(W.parts, W.ids), BP.pack_statics(W.statics, sids)
        g = BO.build_collision_graph(rec, srec, np.asarray(W.ids), np.asarray(sids), float(G["policy"]["dt_max"]),
                                     float(G["policy"]["growth"]))
        want = sw["graph"]
        keys = [tuple(int(x) for x in e) for e in want["edges"]]
        assert list(g.edges) == keys, f"sweep {k}"
        assert np.array_equal(np.array([g.edges[e] for e in keys]).reshape(-1, 2), want["windows"]), f"sweep {k}"
        assert [(int(p), int(s)) for p, ss in g.static_links.items() for s in ss] == \
            [tuple(int(x) for x in l) for l in want["links"]], f"sweep {k}"
        assert np.array_equal(np.array([g.dts[p] for p in W.ids]), want["dts"]), f"sweep {k}"
        n_edges += len(keys)
        bodies = {pid: np.asarray(CT.body_record(p)) for pid, p in W.parts.items()}
        for s in sw["solves"]:
            vel, ang, it, conv, _lam, _fr = CO.solve_impulses(_clist(s["contacts"]), bodies, cfg)
            bids = [int(b) for b in s["bodies"]]
            assert list(vel) == bids and it == int(s["iterations"]) and conv == bool(s["converged"]), f"sweep {k}"
            for j, b in enumerate(bids):
                assert np.array_equal(vel[b], s["velocity"][j]) and np.array_equal(ang[b], s["angular_velocity"][j])
            n_solves += 1
        for cm in sw["commits"]:
            cl = _clist(cm["contacts"])
            mem = [int(m) for m in cm["members"]]
            sol = None
            if bool(cm["has_solution"]):
                b2 = [int(b) for b in cm["sol_bodies"]]
                sol = ({b: cm["sol_velocity"][j] for j, b in enumerate(b2)},
                       {b: cm["sol_angular_velocity"][j] for j, b in enumerate(b2)})
            new = CO.integrate_cluster(mem, float(cm["t_current"]) + float(cm["dt"]), cl, bodies, sol)
            CO.apply_separation(cl, new, {i: bodies[i][CO.B_INVM] for i in mem}, float(cm["beta"]))
            for j, pid in enumerate(mem):
                for q, f in enumerate(("position", "velocity", "rotation", "angular_velocity")):
                    assert np.array_equal(new[pid][q], cm["new"][f][j]), f"sweep {k} member {pid} {f}"
                assert new[pid][4] == cm["new"]["t"][j]
            n_commits += 1
    assert n_edges > 1000 and n_solves >= 20 and n_commits >= 50
