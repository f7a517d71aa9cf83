"""Whole sweeps of the reference engine replayed stage by stage on the GPU.

tests/golden/engine_steps.npz records 40 sweeps of `ltsdem.engine.step`
(engine.py:146-261, "stacks" scenario, 80 particles): per sweep the
timelines, the collision graph the engine got, every `solve_impulses` call
and every commit (`integrate_cluster` + `apply_separation`) with the
members' new snapshots (tests/golden/make_golden_engine.py).  Each stage
goes through the package's drop-in module with the engine's own inputs and
must return what the engine got:

* `broadphase.build_collision_graph`: bit for bit (edges in dict order,
  windows, static links, step bounds);
* `contacts.solve_impulses` / `solve_batch`: bit for bit when no touched
  body spins, else 1e-12 relative (quaternions.advance's sin/cos);
* `contacts.integrate_batch` (the sweep's commits in one launch) and the
  single-cluster `integrate_cluster` + `apply_separation`: same contract.

The narrow-phase stage of the same run is replayed by tests/test_gpu_sweep.py."""

from types import SimpleNamespace as NS

import numpy as np
import pytest

from golden import scene_codec as SC
from helpers import golden

pytestmark = pytest.mark.gpu

RTOL = 1e-12


@pytest.fixture(scope="module")
def W():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_15417_b200 import bodies as B
    from paper_2309_15417_b200 import broadphase, contacts

    G = golden("engine_steps")
    ids = [int(i) for i in G["ids"]]
    parts = {}
    for k, rec in enumerate(G["bodies"]):
        p = SC.decode_body(rec)
        m = 1.0 / float(G["mass"]["inv_mass"][k])
        p.mass = NS(mass=m, inverse_inertia=G["mass"]["inv_inertia"][k].copy())
        p.radius = float(G["spheres"]["radius"][k])
        parts[p.pid] = p
    statics = {}
    for k, rec in enumerate(G["statics"]):
        s = SC.decode_body(rec)
        s.sphere = B.BoundingSphere(center=G["spheres"]["static_center"][k].copy(),
                                    radius=float(G["spheres"]["static_radius"][k]))
        statics[s.sid] = s
    cfg = contacts.SolverConfig(**{k: (int(v) if k == "max_iterations" else float(v))
                                   for k, v in G["solver"].items()})
    return NS(G=G, ids=ids, parts=parts, statics=statics, B=B, BP=broadphase, CT=contacts, cfg=cfg)


def _set_timelines(W, sw):
    for j, pid in enumerate(W.ids):
        tl = W.parts[pid].timeline
        for which in ("old", "current"):
            s = sw[which]
            setattr(tl, which, W.B.state(s["position"][j], s["velocity"][j], s["rotation"][j],
                                         s["angular_velocity"][j], s["t"][j]))
        tl.new = None
        tl.touch()


def _contacts(W, soa):
    from paper_2309_15417_b200.ccd import ContactPoint

    return [ContactPoint(body_a=int(soa["body_a"][i]), body_b=int(soa["body_b"][i]), position=soa["position"][i].copy(),
                         normal=soa["normal"][i].copy(), depth=float(soa["depth"][i]), t=float(soa["t"][i]),
                         tri_a=int(soa["tri_a"][i]), tri_b=int(soa["tri_b"][i]), threshold=float(soa["threshold"][i]))
            for i in range(len(soa["t"]))]


def _spins(W, bids):
    return any(np.any(W.parts[b].timeline.current.angular_velocity != 0.0) for b in bids if b >= 0)


def _same(got, want, exact, what):
    if exact:
        assert np.array_equal(np.asarray(got), np.asarray(want)), what
    else:
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=1e-15, err_msg=what)


def test_collision_graphs_of_the_engine_run(W):
    pol = W.BP.TimeStepPolicy(dt_max=float(W.G["policy"]["dt_max"]), growth=float(W.G["policy"]["growth"]))
    n_edges = 0
    for k, sw in enumerate(W.G["sweeps"]):
        _set_timelines(W, sw)
        g = W.BP.build_collision_graph(W.parts, W.statics, pol)
        want = sw["graph"]
        keys = [tuple(int(x) for x in e) for e in want["edges"]]
        assert list(g.edges) == keys, f"sweep {k}: edges"
        got_w = np.array([g.edges[e] for e in keys]).reshape(-1, 2)
        assert np.array_equal(got_w, want["windows"]), f"sweep {k}: windows"
        links = [(int(p), int(s)) for p, ss in g.static_links.items() for s in ss]
        assert links == [tuple(int(x) for x in l) for l in want["links"]], f"sweep {k}: links"
        assert [int(p) for p in g.static_links] == [int(p) for p in want["link_order"]], f"sweep {k}: link order"
        assert np.array_equal(np.array([g.dts[p] for p in W.ids]), want["dts"]), f"sweep {k}: dts"
        n_edges += len(keys)
    assert n_edges > 1000


def test_impulse_solutions_of_the_engine_run(W):
    n = n_exact = 0
    for k, sw in enumerate(W.G["sweeps"]):
        if not sw["solves"]:
            continue
        _set_timelines(W, sw)
        lists = [_contacts(W, s["contacts"]) for s in sw["solves"]]
        # every call on its own, and (clusters of a sweep are disjoint) all of them in one launch
        singles = [W.CT.solve_impulses(cl, W.parts, W.cfg) for cl in lists]
        batch = W.CT.solve_batch(lists, W.parts, W.cfg)
        for s, one, many in zip(sw["solves"], singles, batch):
            bids = [int(b) for b in s["bodies"]]
            exact = not _spins(W, bids)
            for sol in (one, many):
                assert list(sol.velocities) == bids, f"sweep {k}: solution order"
                assert sol.iterations == int(s["iterations"]) and sol.converged == bool(s["converged"])
                for j, b in enumerate(bids):
                    _same(sol.velocities[b], s["velocity"][j], exact, f"sweep {k} body {b} velocity")
                    _same(sol.angular_velocities[b], s["angular_velocity"][j], exact, f"sweep {k} body {b} spin")
            n += 1
            n_exact += exact
    assert n >= 20 and n_exact >= 1


def _commit_inputs(W, c):
    cluster = NS(members=tuple(int(m) for m in c["members"]), t_current=float(c["t_current"]), dt=float(c["dt"]))
    contacts = _contacts(W, c["contacts"])
    result = NS(dt=float(c["dt"]), contacts=contacts)
    sol = None
    if bool(c["has_solution"]):
        bids = [int(b) for b in c["sol_bodies"]]
        sol = NS(velocities={b: c["sol_velocity"][j] for j, b in enumerate(bids)},
                 angular_velocities={b: c["sol_angular_velocity"][j] for j, b in enumerate(bids)})
    return cluster, result, sol


def _check_new(W, c, k, label):
    exact = not _spins(W, [int(m) for m in c["members"]])
    for j, pid in enumerate(int(m) for m in c["members"]):
        s = W.parts[pid].timeline.new
        assert s is not None, f"sweep {k}: member {pid} has no new snapshot"
        for f in ("position", "velocity", "rotation", "angular_velocity"):
            _same(getattr(s, f), c["new"][f][j], exact, f"{label} sweep {k} member {pid} {f}")
        _same(s.t, c["new"]["t"][j], True, f"{label} sweep {k} member {pid} t")
    return exact


def test_commits_of_the_engine_run(W):
    n = n_exact = 0
    for k, sw in enumerate(W.G["sweeps"]):
        if not sw["commits"]:
            continue
        ins = [_commit_inputs(W, c) for c in sw["commits"]]
        beta = float(sw["commits"][0]["beta"])
        # the sweep's commits in one launch, as a sweep driver would issue them
        _set_timelines(W, sw)
        W.CT.integrate_batch([i[0] for i in ins], W.parts, [i[1] for i in ins], [i[2] for i in ins], beta=beta)
        for c in sw["commits"]:
            n_exact += _check_new(W, c, k, "batch")
            n += 1
        # and cluster by cluster through the reference's two calls (engine.py:227-228)
        if k % 4 == 0:
            _set_timelines(W, sw)
            for c, (cluster, result, sol) in zip(sw["commits"], ins):
                W.CT.integrate_cluster(cluster, W.parts, result, sol)
                W.CT.apply_separation(result.contacts, W.parts, beta)
                _check_new(W, c, k, "single")
    assert n >= 50 and n_exact >= 1
