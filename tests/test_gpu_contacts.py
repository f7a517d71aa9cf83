"""GPU parity of the contact consumers (ltsg_solve_impulses / ltsg_integrate).

Against the reference's own outputs (tests/golden/contacts.npz, produced by
ltsdem.contacts: solve_impulses contacts.py:114-198, color_contact_graph
:58-78, integrate_cluster :225-253, apply_separation :256-285): bit for bit
for bodies without spin; spinning bodies (quaternions.advance's sin/cos)
within 1e-12 relative.  And through the drop-in object API against the
pinned oracle.
"""

from types import SimpleNamespace as NS

import numpy as np
import pytest

from helpers import golden
from oracle import contact_oracle as CO
from test_contact_oracle import case_inputs

pytestmark = pytest.mark.gpu


def _cs():
    from paper_2309_15417_b200 import contacts as CS

    return CS


def _arrays(g):
    ids = [int(i) for i in g["ids"]]
    index = {b: k for k, b in enumerate(ids)}
    side = np.array([[index.get(int(a), -1) if a >= 0 else -1, index.get(int(b), -1) if b >= 0 else -1]
                     for a, b in zip(g["body_a"], g["body_b"])], dtype=np.int32).reshape(-1, 2)
    idp = np.stack([g["body_a"], g["body_b"]], axis=1).astype(np.int64).reshape(-1, 2)
    return ids, index, side, idp


def _close(got, ref, spin, what):
    if spin:
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13, err_msg=what)
    else:
        np.testing.assert_array_equal(got, ref, err_msg=what)


@pytest.mark.parametrize("name", [g["name"] for g in golden("contacts")["cases"]])
def test_solve_and_integrate_match_the_reference(name):
    CS = _cs()
    g = next(c for c in golden("contacts")["cases"] if c["name"] == name)
    ids, index, side, idp = _arrays(g)
    cfg = CS.SolverConfig(**{k: g["cfg"][k] for k in ("restitution", "friction", "relaxation", "penalty",
                                                      "threshold", "max_iterations", "beta")})
    n_c = len(g["t"])
    off = np.array([0, n_c], dtype=np.int64)
    r = CS.solve_arrays(g["rec"], side, g["position"], g["normal"], g["t"], off, cfg)
    spin = bool(g["spin"])
    if not spin:
        assert int(r["iterations"][0]) == g["iterations"] and bool(r["converged"][0]) == g["converged"]
    np.testing.assert_array_equal(r["color"], g["color"])
    sol = [index[int(b)] for b in g["sol_ids"]]
    assert set(np.flatnonzero(r["touched"])) == set(sol)
    _close(r["velocity"][sol], g["sol_vel"], spin, "velocities")
    _close(r["angular_velocity"][sol], g["sol_ang"], spin, "angular velocities")
    _close(r["normal_impulse"], g["lam"], spin, "normal impulses")
    _close(r["friction_impulse"], g["fric"].reshape(-1, 3), spin, "friction impulses")
    member = np.arange(len(ids), dtype=np.int32)
    new = CS.integrate_arrays(g["rec"], np.array([0, len(ids)]), member, np.array([g["t_current"] + g["dt"]]), off,
                              side, idp, g["normal"], g["t"], g["depth"], r["velocity"], r["angular_velocity"],
                              r["touched"].astype(np.int32) if n_c else None, cfg.beta, separate=True)
    _close(new, g["new"], spin, "new snapshots")


def test_batched_launch_equals_single_launches():
    """Every non-spinning golden cluster with the default configuration in
    one ltsg_solve_impulses call (one warp per cluster): identical to the
    single-cluster calls, bit for bit."""
    CS = _cs()
    cases = [g for g in golden("contacts")["cases"] if not g["spin"] and len(g["t"])]
    cfg = CS.SolverConfig(threshold=1e-9, max_iterations=64)
    recs, sides, pos, nrm, tt, off = [], [], [], [], [], [0]
    base = 0
    singles = []
    for g in cases:
        ids, index, side, idp = _arrays(g)
        singles.append(CS.solve_arrays(g["rec"], side, g["position"], g["normal"], g["t"],
                                       np.array([0, len(g["t"])]), cfg))
        recs.append(g["rec"])
        sides.append(np.where(side >= 0, side + base, -1))
        pos.append(g["position"]), nrm.append(g["normal"]), tt.append(g["t"])
        off.append(off[-1] + len(g["t"]))
        base += len(ids)
    r = CS.solve_arrays(np.concatenate(recs), np.concatenate(sides).astype(np.int32), np.concatenate(pos),
                        np.concatenate(nrm), np.concatenate(tt), np.array(off), cfg)
    base = 0
    for k, (g, s) in enumerate(zip(cases, singles)):
        nb = len(g["ids"])
        assert r["iterations"][k] == s["iterations"][0] and r["converged"][k] == s["converged"][0]
        np.testing.assert_array_equal(r["velocity"][base:base + nb][s["touched"]], s["velocity"][s["touched"]])
        np.testing.assert_array_equal(r["normal_impulse"][off[k]:off[k + 1]], s["normal_impulse"])
        base += nb


def _objects(g):
    """Package-side particle objects carrying a golden case's records (mass
    chosen so that 1 / mass reproduces the record's inverse mass)."""
    from paper_2309_15417_b200 import bodies as B

    parts = {}
    for i, r in zip(g["ids"], g["rec"]):
        m = 1.0 / r[14]
        assert 1.0 / m == r[14]
        st = B.state(r[0:3], velocity=r[3:6], rotation=r[6:10], angular_velocity=r[10:13], t=r[13])
        p = B.Particle(pid=int(i), tree=None, epsilon=0.01, radius=1.0, timeline=B.timeline(st))
        p.mass = NS(mass=m, inverse_inertia=r[15:24].reshape(3, 3).copy())
        parts[int(i)] = p
    from paper_2309_15417_b200.ccd import ContactPoint

    contacts = [ContactPoint(body_a=int(a), body_b=int(b), position=p.copy(), normal=n.copy(), depth=float(d),
                             t=float(t)) for a, b, p, n, t, d in zip(g["body_a"], g["body_b"], g["position"],
                                                                       g["normal"], g["t"], g["depth"])]
    return parts, contacts


@pytest.mark.parametrize("name", ["two_impacts", "random_1", "random_8", "large"])
def test_object_api_matches_the_oracle(name):
    CS = _cs()
    g = next(c for c in golden("contacts")["cases"] if c["name"] == name)
    parts, contacts = _objects(g)
    cfg = CS.SolverConfig(**{k: g["cfg"][k] for k in ("restitution", "friction", "relaxation", "penalty",
                                                      "threshold", "max_iterations", "beta")})
    sol = CS.solve_impulses(contacts, parts, cfg)
    bodies, ocon = case_inputs(g)
    vel, ang, iters, conv, lam, fric = CO.solve_impulses(ocon, bodies, g["cfg"])
    assert list(sol.velocities) == list(vel) and sol.iterations == iters and sol.converged == conv
    for b in vel:
        np.testing.assert_array_equal(sol.velocities[b], vel[b])
        np.testing.assert_array_equal(sol.angular_velocities[b], ang[b])
    assert sol.normal_impulses == lam
    cluster = NS(members=tuple(int(i) for i in g["ids"]), t_current=g["t_current"], dt=g["dt"])
    result = NS(dt=g["dt"], contacts=contacts)
    CS.integrate_cluster(cluster, parts, result, sol)
    CS.apply_separation(contacts, parts, cfg.beta)
    for k, i in enumerate(g["ids"]):
        s = parts[int(i)].timeline.new
        got = np.concatenate([s.position, s.velocity, s.rotation, s.angular_velocity, [s.t]])
        np.testing.assert_array_equal(got, g["new"][k])
        assert parts[int(i)].timeline.version >= 1


def test_empty_and_validation():
    CS = _cs()
    assert CS.solve_impulses([], {}).converged
    with pytest.raises(ValueError):
        CS.SolverConfig(restitution=1.5)
    g = next(c for c in golden("contacts")["cases"] if c["name"] == "head_on")
    parts, contacts = _objects(g)
    contacts[0].t = -1.0  # before the bodies' current snapshot: the reference's free flight raises
    with pytest.raises(ValueError):
        CS.solve_impulses(contacts, parts)
