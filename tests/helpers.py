"""Shared test helpers: fixture loading, scene decoding, result comparison."""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
sys.path.insert(0, GOLDEN)

import gio  # noqa: E402
import scene_codec as SC  # noqa: E402

_cache = {}


def golden(name):
    if name not in _cache:
        _cache[name] = gio.load(os.path.join(GOLDEN, f"{name}.npz"))
    return _cache[name]


def scene_inputs(case):
    """Decode a fixture scene into (particles, statics, pairs, cluster)."""
    bodies = [SC.decode_body(b) for b in case["bodies"]]
    particles = {b.pid: b for b in bodies if hasattr(b, "timeline")}
    statics = {b.sid: b for b in bodies if not hasattr(b, "timeline")}
    pairs = [(int(a), int(b)) for a, b in case["pairs"]]
    cluster = SimpleNamespace(dt=case["dt"], t_current=case["t_base"])
    return particles, statics, pairs, cluster


def run_case(api, case, exhaustive=None):
    """Run one fixture scene through an API module exposing the reference
    call surface (the oracle, or the GPU package)."""
    particles, statics, pairs, cluster = scene_inputs(case)
    ex = case["exhaustive"] if exhaustive is None else exhaustive
    if case["mode"] == "pair":
        # pair mode keeps the fixture's body order: bodies[0] is body_a
        ba = SC.decode_body(case["bodies"][0])
        bb = SC.decode_body(case["bodies"][1])
        return api.pair_earliest_contact(ba, bb, case["dt"], widen=case["widen"], exhaustive=ex)
    return api.compute_effective_dt(cluster, particles, statics, pairs, widen=case["widen"])


def contacts_soa(contacts):
    return SC.encode_contacts(contacts)


def compare_contacts(got, want, *, rtol=0.0, atol=0.0, label=""):
    """Field-by-field contact comparison; exact when rtol == atol == 0."""
    g = got if isinstance(got, dict) else contacts_soa(got)
    assert len(g["t"]) == len(want["t"]), f"{label}: {len(g['t'])} contacts vs {len(want['t'])}"
    for f in ("body_a", "body_b", "tri_a", "tri_b"):
        np.testing.assert_array_equal(g[f], want[f], err_msg=f"{label}: {f}")
    for f in ("position", "normal", "depth", "t", "threshold"):
        if rtol == 0.0 and atol == 0.0:
            np.testing.assert_array_equal(g[f], want[f], err_msg=f"{label}: {f}")
        else:
            np.testing.assert_allclose(g[f], want[f], rtol=rtol, atol=atol, err_msg=f"{label}: {f}")


def compare_result(res, want, *, exact=True, tau_tol=1e-9, rtol=1e-9, atol=1e-12, label="",
                   raw=None):
    """Compare a NarrowResult-like object with a fixture result."""
    assert res.collision == want["collision"], f"{label}: collision"
    assert res.narrowing_iters == want["narrowing_iters"], f"{label}: narrowing_iters"
    assert len(res.bound_history) == len(want["bound_history"]), f"{label}: bound_history"
    if exact:
        assert res.dt == want["dt"], f"{label}: dt {res.dt!r} vs {want['dt']!r}"
        assert res.first_contact == want["first_contact"], f"{label}: first_contact"
        np.testing.assert_array_equal(np.array(res.bound_history, float), want["bound_history"])
        if raw is not None:
            compare_contacts(raw, want["raw"], label=label + " raw")
        compare_contacts(res.contacts, want["contacts"], label=label + " fused")
    else:
        assert abs(res.dt - want["dt"]) <= tau_tol * (1 + abs(want["dt"])), f"{label}: dt"
        if want["first_contact"] is None:
            assert res.first_contact is None
        else:
            assert abs(res.first_contact - want["first_contact"]) <= tau_tol, f"{label}: first"
        if raw is not None:
            compare_contacts(raw, want["raw"], rtol=rtol, atol=max(atol, tau_tol),
                             label=label + " raw")
        compare_contacts(res.contacts, want["contacts"], rtol=rtol, atol=max(atol, tau_tol),
                         label=label + " fused")
