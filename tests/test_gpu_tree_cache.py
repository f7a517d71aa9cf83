"""The public API's device-resident tree cache (ccd.DeviceScene cache_trees):
results with the cache equal results without it, state changes between calls
are seen, a different tree set re-uploads, and a cached call copies only the
per-step arrays."""

import numpy as np
import pytest

from oracle import narrow_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ccd():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_15417_b200 import ccd

    yield ccd
    ccd.set_tree_cache(True)


def _same(a, b):
    assert np.array_equal(a.dt, b.dt) and np.array_equal(a.collision, b.collision)
    assert np.array_equal(a.fused_offset, b.fused_offset)
    for k in a.contacts:
        assert np.array_equal(a.contacts[k], b.contacts[k]), k


def test_cached_equals_uncached_and_sees_state_changes(ccd):
    from paper_2309_15417_b200 import scenes

    sc = scenes.config4(n_pairs=6, subdiv=1)
    pairs = [(sc.body(a), sc.body(b)) for a, b in sc.pairs]
    ccd.set_tree_cache(False)
    cold = ccd.earliest_contacts(pairs, sc.dt)
    ccd.set_tree_cache(True)
    tm = {}
    first = ccd.earliest_contacts(pairs, sc.dt, timings=tm)
    tm2 = {}
    warm = ccd.earliest_contacts(pairs, sc.dt, timings=tm2)
    _same(cold, first)
    _same(cold, warm)
    assert tm2["h2d_bytes"][0] < tm["h2d_bytes"][0] // 10  # states and pair tables only
    # move every body: the cached geometry must be combined with the new states
    for b in {id(x): x for p in pairs for x in p}.values():
        st = b.timeline.current
        st.position = np.asarray(st.position) + np.array([0.013, -0.007, 0.002])
        st.velocity = -np.asarray(st.velocity)
    moved = ccd.earliest_contacts(pairs, sc.dt)
    for k, (a, b) in enumerate(pairs):
        got = moved.result(k)
        ref = O.pair_earliest_contact(a, b, sc.dt[k])
        assert got.collision == ref.collision
        assert abs(got.dt - ref.dt) <= 1e-9
        assert len(got.contacts) == len(ref.contacts)


def test_new_tree_set_reuploads(ccd):
    from paper_2309_15417_b200 import scenes

    ccd.set_tree_cache(True)
    s1 = scenes.config1(n_pairs=2, subdiv=1)
    s2 = scenes.config1(n_pairs=3, subdiv=2, seed_offset=7)
    p1 = [(s1.body(a), s1.body(b)) for a, b in s1.pairs]
    p2 = [(s2.body(a), s2.body(b)) for a, b in s2.pairs]
    ccd.earliest_contacts(p1, s1.dt)
    tm = {}
    r2 = ccd.earliest_contacts(p2, s2.dt, timings=tm)
    assert tm["h2d_bytes"][0] > 100_000  # the new trees travelled
    for k, (a, b) in enumerate(p2):
        got = r2.result(k)
        ref = O.pair_earliest_contact(a, b, s2.dt[k])
        assert got.dt == ref.dt and len(got.contacts) == len(ref.contacts)
        for x, y in zip(got.contacts, ref.contacts):
            assert np.array_equal(x.position, y.position)
