"""The drop-in claim with genuine reference objects: `ltsdem.body.make_particle`
/ `make_static` particles and `ltsdem.clustering.Cluster` are packed exactly
like the package's duck-typed classes built from the same data.  Needs the
reference importable (this build container); skipped where it is absent
(the GPU box)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference not present on this host", allow_module_level=True)
sys.path.insert(0, REF)

from golden import scene_codec as SC  # noqa: E402
from paper_2309_15417_b200 import packing, scenes  # noqa: E402
from paper_2309_15417_b200.ccd import _cluster_problem, _pair_problem  # noqa: E402


def _ref_world():
    from ltsdem.body import initial_state, make_particle, make_static
    from ltsdem.clustering import Cluster
    from ltsdem.mesh import TriangleMesh, make_plane

    rng = np.random.default_rng(3)
    parts = {}
    for pid, sub in enumerate((2, 1, 0)):
        v, f = scenes.icosphere(sub)
        v = v * (1 + rng.uniform(-0.05, 0.05, len(v)))[:, None]
        parts[pid] = make_particle(pid, TriangleMesh(v, f), 1e-3, initial_state(
            position=rng.normal(size=3), velocity=rng.normal(size=3),
            rotation=scenes.random_quaternions(rng, 1)[0], angular_velocity=rng.normal(size=3)))
    v, f = scenes.box((0.3, 0.2, 0.1))
    parts[3] = make_particle(3, TriangleMesh(v, f), 1e-3, initial_state(position=(0.0, 0.0, 1.0)))
    floor = make_static(-1, make_plane((-3.0, -3.0, -2.0), (3.0, 3.0, -2.0)), epsilon=1e-3)
    cluster = Cluster(members=(0, 1, 2, 3), t_current=0.5, dt=0.05)
    pairs = [(0, 1), (1, 2), (0, 3), (2, -1), (3, -1)]
    return parts, {-1: floor}, cluster, pairs


def _decoded(parts, statics):
    dp = {k: SC.decode_body(SC.encode_body(b)) for k, b in parts.items()}
    ds = {k: SC.decode_body(SC.encode_body(b)) for k, b in statics.items()}
    return dp, ds


def _assert_same_scene(a, b):
    xa, xb = a.arrays(), b.arrays()
    assert sorted(xa) == sorted(xb)
    for k in xa:
        va, vb = np.asarray(xa[k]), np.asarray(xb[k])
        assert va.dtype == vb.dtype and va.shape == vb.shape, k
        assert va.tobytes() == vb.tobytes(), k
    assert a.records().tobytes() == b.records().tobytes()


def test_cluster_of_reference_objects_packs_like_duck_types():
    parts, statics, cluster, pairs = _ref_world()
    dp, ds = _decoded(parts, statics)
    got = packing.pack([_cluster_problem(cluster, parts, statics, pairs)])
    want = packing.pack([_cluster_problem(cluster, dp, ds, pairs)])
    _assert_same_scene(got, want)
    # the cluster fields the path reads (ccd.py:505-524)
    assert got.arrays()["problem_dt"][0] == cluster.dt
    assert got.arrays()["problem_tbase"][0] == cluster.t_current


def test_pairs_of_reference_objects_pack_like_duck_types():
    parts, statics, _, _ = _ref_world()
    dp, ds = _decoded(parts, statics)
    probs_ref = [_pair_problem(parts[0], parts[1], 0.1), _pair_problem(parts[2], statics[-1], 0.0),
                 _pair_problem(parts[3], parts[3], 0.2)]
    probs_dt = [_pair_problem(dp[0], dp[1], 0.1), _pair_problem(dp[2], ds[-1], 0.0),
                _pair_problem(dp[3], dp[3], 0.2)]
    _assert_same_scene(packing.pack(probs_ref), packing.pack(probs_dt))
    # the batched fast path (pinned Packer, C helper) too
    pk = packing.Packer(pinned=False)
    a = pk.pack_pairs([(parts[0], parts[1]), (parts[2], statics[-1])], np.array([0.1, 0.0]))
    pk2 = packing.Packer(pinned=False)
    b = pk2.pack_pairs([(dp[0], dp[1]), (dp[2], ds[-1])], np.array([0.1, 0.0]))
    _assert_same_scene(a, b)
