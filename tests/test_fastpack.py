"""The C packing helpers (csrc/fastpack.c): the gathered state table equals
packing.body_state_row for dynamic and static bodies, whatever the field
types; the identity checks of the pair list and tree set."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2309_15417_b200 import packing


@pytest.fixture(scope="module")
def fp():
    if packing._fastpack is None:
        pytest.skip("packing helper not built")
    return packing._fastpack


def _body(rng, kind):
    if kind == "static":
        return SimpleNamespace(sid=-1, tree=object())
    st = SimpleNamespace(position=rng.normal(size=3), velocity=rng.normal(size=3),
                         rotation=rng.normal(size=4), angular_velocity=rng.normal(size=3))
    if kind == "list":  # plain sequences instead of arrays
        st.position = list(st.position)
        st.rotation = tuple(st.rotation)
    if kind == "strided":  # a non-contiguous view
        st.velocity = np.arange(6.0)[::2] * 0.5
    return SimpleNamespace(pid=1, tree=object(), timeline=SimpleNamespace(current=st))


def test_gather_states_matches_rows(fp):
    rng = np.random.default_rng(3)
    bodies = [_body(rng, k) for k in ("array", "static", "list", "strided", "array", "static")]
    out = np.full((len(bodies), 16), np.nan)
    fp.gather_states(bodies, out)
    want = np.stack([packing.body_state_row(b) for b in bodies])
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))


def test_gather_states_rejects_bad_fields(fp):
    rng = np.random.default_rng(4)
    b = _body(rng, "array")
    b.timeline.current.position = np.zeros(2)
    with pytest.raises(ValueError):
        fp.gather_states([b], np.zeros((1, 16)))
    with pytest.raises(ValueError):
        fp.gather_states([_body(rng, "array")], np.zeros((2, 16)))


def test_identity_checks(fp):
    rng = np.random.default_rng(5)
    bodies = [_body(rng, "array") for _ in range(4)]
    pairs = [(bodies[0], bodies[1]), (bodies[2], bodies[3])]
    flat = [bodies[0], bodies[1], bodies[2], bodies[3]]
    assert fp.pairs_are(pairs, flat)
    assert not fp.pairs_are([(bodies[1], bodies[0]), pairs[1]], flat)
    assert not fp.pairs_are(pairs[:1], flat)
    trees = [b.tree for b in bodies]
    assert fp.trees_are(bodies, trees)
    bodies[2].tree = object()
    assert not fp.trees_are(bodies, trees)
