"""The contact-consumer CPU oracle against the reference's own outputs.

tests/golden/contacts.npz was produced by running the reference's
`ltsdem.contacts` (solve_impulses contacts.py:114-198, color_contact_graph
:58-78, integrate_cluster :225-253, apply_separation :256-285) on seeded
clusters (tests/golden/make_golden_contacts.py).  The oracle must reproduce
every output bit for bit.
"""

import numpy as np
import pytest

from helpers import golden
from oracle import contact_oracle as CO


def _cases():
    return golden("contacts")["cases"]


def case_inputs(g):
    bodies = {int(i): r for i, r in zip(g["ids"], g["rec"])}
    contacts = [{"body_a": int(a), "body_b": int(b), "position": p, "normal": n, "t": float(t), "depth": float(d)}
                for a, b, p, n, t, d in zip(g["body_a"], g["body_b"], g["position"], g["normal"], g["t"],
                                            g["depth"])]
    return bodies, contacts


@pytest.mark.parametrize("name", [g["name"] for g in golden("contacts")["cases"]])
def test_oracle_solve_and_integrate_bit_exact(name):
    g = next(c for c in _cases() if c["name"] == name)
    bodies, contacts = case_inputs(g)
    vel, ang, iters, conv, lam, fric = CO.solve_impulses(contacts, bodies, g["cfg"])
    assert iters == g["iterations"] and conv == g["converged"]
    assert list(vel) == [int(i) for i in g["sol_ids"]]
    np.testing.assert_array_equal(np.array(list(vel.values())).reshape(-1, 3), g["sol_vel"])
    np.testing.assert_array_equal(np.array(list(ang.values())).reshape(-1, 3), g["sol_ang"])
    np.testing.assert_array_equal(np.array(lam), g["lam"])
    np.testing.assert_array_equal(np.array(fric).reshape(-1, 3), g["fric"])
    classes = CO.color_contact_graph([(c["body_a"], c["body_b"]) for c in contacts])
    col = np.zeros(len(contacts), dtype=np.int64)
    for k, cl in enumerate(classes):
        col[cl] = k
    np.testing.assert_array_equal(col, g["color"])
    members = [int(i) for i in g["ids"]]
    new = CO.integrate_cluster(members, g["t_current"] + g["dt"], contacts, bodies,
                               (vel, ang) if contacts else None)
    CO.apply_separation(contacts, new, {i: bodies[i][CO.B_INVM] for i in members}, g["cfg"]["beta"])
    got = np.array([np.concatenate([new[i][0], new[i][1], new[i][2], new[i][3], [new[i][4]]]) for i in members])
    np.testing.assert_array_equal(got, g["new"])


def test_fixtures_cover_both_regimes():
    cs = _cases()
    assert any(not c["converged"] for c in cs) and any(c["converged"] for c in cs)
    assert any(c["spin"] for c in cs) and any(len(c["t"]) >= 100 for c in cs)
    assert any((c["body_b"] < 0).any() for c in cs)
