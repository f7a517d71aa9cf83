"""The guided pre-decision of static generations (k_guide_static,
csrc/bound32.cuh) must never change a result: it only decides rows through
an exact single-feature witness (ccd.py:153: the reference takes the minimum
over 15 features) or a certified separating direction, and hands everything
else to the exact 15-feature kernel.

* guide on vs `LTSG_NO_GUIDE=1`: every output array identical, bit for bit,
  on the static BASELINE-shaped scenes, in both traversal modes;
* against the CPU oracle on scenes built to stress the guide: scaled by
  1e-6 .. 1e6 and moved 1e6 away from the origin (the FP32 guide runs in a
  local frame), flat slivers and zero-area triangles (never culled),
  deeply interpenetrating bodies (distance 0 rows), exactly touching boxes;
* the counters show the guide really ran (rows_bound > 0)."""

import numpy as np
import pytest

from golden import scene_codec as SC
from helpers import compare_contacts
from oracle import narrow_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_15417_b200 import ccd

    return ccd


def _canonical(soa):
    """Raw records in the fusion sort order (ccd.py:541-542), as the GPU emits them."""
    if len(soa["t"]) == 0:
        return soa
    r9 = lambda x: np.rint(x * 1e9) / 1e9  # noqa: E731
    pos = soa["position"]
    order = np.lexsort((soa["tri_b"], soa["tri_a"], r9(pos[:, 2]), r9(pos[:, 1]), r9(pos[:, 0]),
                        soa["t"], soa["body_b"], soa["body_a"]))
    return {k: v[order] for k, v in soa.items()}


def _same_batch(a, b, label):
    for f in ("dt", "collision", "first_contact", "fused_offset"):
        x, y = getattr(a, f), getattr(b, f)
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)), (label, f)
    for soa_a, soa_b, what in ((a.contacts, b.contacts, "fused"), (a.raw, b.raw, "raw")):
        assert set(soa_a) == set(soa_b)
        for k in soa_a:
            x, y = np.ascontiguousarray(soa_a[k]), np.ascontiguousarray(soa_b[k])
            assert x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8)), (label, what, k)


@pytest.mark.parametrize("config,kwargs,exhaustive", [
    ("c1", dict(n_pairs=48, subdiv=2), False),
    ("c1", dict(n_pairs=6, subdiv=2), True),
    ("c2", dict(n_boxes=200), False),
    ("c3", dict(n_rocks=300), False),
], ids=["c1", "c1-exhaustive", "c2", "c3"])
def test_guide_on_equals_guide_off(G, monkeypatch, config, kwargs, exhaustive):
    from paper_2309_15417_b200 import scenes

    scene = scenes.CONFIGS[config](**kwargs)
    pairs = [(scene.body(a), scene.body(b)) for a, b in scene.pairs]
    runs = {}
    for mode in ("on", "off"):
        if mode == "off":
            monkeypatch.setenv("LTSG_NO_GUIDE", "1")
        else:
            monkeypatch.delenv("LTSG_NO_GUIDE", raising=False)
        # twice: the first call on a scene runs the synchronous traversal, the second the asynchronous one
        runs[mode] = [G.earliest_contacts(pairs, scene.dt, raw=True, exhaustive=exhaustive) for _ in range(2)]
    for k in range(2):
        _same_batch(runs["on"][k], runs["off"][k], f"{config} call {k}")
    on, off = runs["on"][1].stats, runs["off"][1].stats
    assert on["rows_screen"] == off["rows_screen"]
    assert on["rows_bound"] > 0 and off["rows_bound"] == 0
    assert on["rows_bound"] + on["rows_screen_exact"] == off["rows_screen_exact"]


def _icosphere_particle(pid, sub, scale, centre, eps, rng, squash=None, q=None):
    from paper_2309_15417_b200 import bodies as B
    from paper_2309_15417_b200 import scenes

    v, f = scenes.icosphere(sub)
    v = v * (1.0 + rng.uniform(-0.05, 0.05, size=len(v)))[:, None]
    if squash is not None:
        v = v * np.asarray(squash)[None, :]
    v = v * scale
    c = v - B.centre_of_mass(v, f)
    corners = np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1)
    tree = scenes.build_trees([corners], eps)[0]
    rot = scenes.random_quaternions(rng, 1)[0] if q is None else q
    return B.make_particle(pid, v, f, eps, B.state(centre, rotation=rot), tree=tree)


def _check_pairs_vs_oracle(G, pairs, label):
    batch = G.earliest_contacts(pairs, 0.0, raw=True)
    assert batch.stats["rows_bound"] > 0, label
    for k, (a, b) in enumerate(pairs):
        ref = O.pair_earliest_contact(a, b, 0.0)
        got = batch.result(k)
        assert got.dt == ref.dt and got.collision == ref.collision, (label, k)
        compare_contacts(got.contacts, SC.encode_contacts(ref.contacts), label=f"{label} pair {k}")
        compare_contacts(_canonical(SC.encode_contacts(batch.raw_contacts(k))), _canonical(SC.encode_contacts(ref.raw)),
                         label=f"{label} raw pair {k}")


@pytest.mark.parametrize("scale", [1e-6, 1e-3, 1.0, 1e3, 1e6], ids=lambda s: f"scale{s:g}")
def test_scaled_and_shifted_scenes_vs_oracle(G, scale):
    """The same near-touching pairs at sizes 1e-6 .. 1e6, 1e6 body sizes away
    from the origin: the guide's FP32 frame is local to each row."""
    rng = np.random.default_rng(int(np.log10(scale)) + 20)
    pairs = []
    for k in range(6):
        far = rng.normal(size=3) * 1e6 * scale
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        gap = rng.uniform(1.9, 2.1) * scale
        a = _icosphere_particle(2 * k, 2, scale, far - 0.5 * gap * axis, 0.01 * scale, rng)
        b = _icosphere_particle(2 * k + 1, 2, scale, far + 0.5 * gap * axis, 0.01 * scale, rng)
        pairs.append((a, b))
    _check_pairs_vs_oracle(G, pairs, f"scale {scale:g}")


def test_slivers_and_flat_bodies_vs_oracle(G):
    """Bodies squashed to 1e-4 and 1e-9 of their size: needle and sliver
    triangles, which the culls never touch, against round ones."""
    rng = np.random.default_rng(7)
    pairs = []
    for k, squash in enumerate([(1.0, 1.0, 1e-4), (1.0, 1e-4, 1.0), (1.0, 1.0, 1e-9), (1e-4, 1e-4, 1.0)]):
        a = _icosphere_particle(2 * k, 2, 1.0, (0.0, 0.0, 0.0), 0.01, rng, squash=squash,
                                q=np.array([1.0, 0.0, 0.0, 0.0]))
        b = _icosphere_particle(2 * k + 1, 2, 0.5, (0.3, 0.2, 0.1), 0.01, rng)
        pairs.append((a, b))
    _check_pairs_vs_oracle(G, pairs, "slivers")


def test_interpenetrating_and_touching_vs_oracle(G):
    """Deep overlap (many rows at distance 0) and boxes that touch exactly
    (face on face, edge on edge: distance exactly equal to the threshold
    minus the halos)."""
    from paper_2309_15417_b200 import bodies as B
    from paper_2309_15417_b200 import scenes

    rng = np.random.default_rng(9)
    pairs = []
    for k, off in enumerate([0.0, 0.3, 1.2]):
        a = _icosphere_particle(2 * k, 2, 1.0, (0.0, 0.0, 0.0), 0.01, rng)
        b = _icosphere_particle(2 * k + 1, 2, 1.0, (off, 0.05, -0.02), 0.01, rng)
        pairs.append((a, b))
    v, f = scenes.box((1.0, 1.0, 1.0))
    c = v - B.centre_of_mass(v, f)
    corners = np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1)
    eps = 1e-3
    tree = scenes.build_trees([corners], eps)[0]
    ident = np.array([1.0, 0.0, 0.0, 0.0])
    for k, pos in enumerate([(1.0, 0.0, 0.0), (1.0 + 2 * eps, 0.0, 0.0), (1.0, 1.0, 0.0), (1.0, 1.0, 1.0),
                             (1.0 + 2 * eps + 1e-9, 0.0, 0.0), (1.0 + 2 * eps + 2e-9, 0.25, 0.5)]):
        a = B.make_particle(100 + 2 * k, v, f, eps, B.state((0.0, 0.0, 0.0), rotation=ident), tree=tree)
        b = B.make_particle(101 + 2 * k, v, f, eps, B.state(pos, rotation=ident), tree=tree)
        pairs.append((a, b))
    _check_pairs_vs_oracle(G, pairs, "overlap/touch")


def test_guide_on_equals_guide_off_random_poses(G, monkeypatch):
    """400 random body pairs (icospheres, rocks and boxes of random size,
    halo and pose; separated, grazing and deeply overlapping) in one batch:
    guide on and off give identical arrays."""
    from paper_2309_15417_b200 import bodies as B
    from paper_2309_15417_b200 import scenes

    rng = np.random.default_rng(2309)
    protos = []
    for sub in (0, 1, 2):
        protos.append(scenes.icosphere(sub))
    for _ in range(3):
        protos.append(scenes.rock(rng))
    protos.append(scenes.box((1.0, 0.6, 0.3)))
    corners, eps_list, spec = [], [], []
    for k in range(800):
        v, f = protos[int(rng.integers(len(protos)))]
        v = v * float(np.exp(rng.uniform(np.log(0.2), np.log(3.0))))
        eps = float(10.0 ** rng.uniform(-4, -1.5))
        c = v - B.centre_of_mass(v, f)
        corners.append(np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1))
        eps_list.append(eps)
        spec.append((v, f, eps))
    trees = scenes.build_trees(corners, eps_list)
    quats = scenes.random_quaternions(rng, 800)
    pairs = []
    for k in range(400):
        (va, fa, ea), (vb, fb, eb) = spec[2 * k], spec[2 * k + 1]
        ra = float(np.linalg.norm(corners[2 * k].reshape(-1, 3), axis=1).max())
        rb = float(np.linalg.norm(corners[2 * k + 1].reshape(-1, 3), axis=1).max())
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        dist = (ra + rb) * float(rng.choice([0.0, 0.3, 0.7, 0.95, 1.0, 1.02, 1.3]))
        base = rng.normal(size=3) * 10.0
        a = B.make_particle(2 * k, va, fa, ea, B.state(base, rotation=quats[2 * k]), tree=trees[2 * k])
        b = B.make_particle(2 * k + 1, vb, fb, eb, B.state(base + dist * axis, rotation=quats[2 * k + 1]),
                            tree=trees[2 * k + 1])
        pairs.append((a, b))
    runs = {}
    for mode in ("on", "off"):
        if mode == "off":
            monkeypatch.setenv("LTSG_NO_GUIDE", "1")
        else:
            monkeypatch.delenv("LTSG_NO_GUIDE", raising=False)
        runs[mode] = [G.earliest_contacts(pairs, 0.0, raw=True) for _ in range(2)]
    for k in range(2):
        _same_batch(runs["on"][k], runs["off"][k], f"random poses call {k}")
    assert runs["on"][1].stats["rows_bound"] > 0
    assert len(runs["on"][1].raw["t"]) > 1000  # the batch really produces contacts
    # and a sample of the pairs against the oracle
    for k in rng.choice(400, size=12, replace=False):
        a, b = pairs[int(k)]
        ref = O.pair_earliest_contact(a, b, 0.0)
        got = runs["on"][1].result(int(k))
        assert got.dt == ref.dt and got.collision == ref.collision
        compare_contacts(got.contacts, SC.encode_contacts(ref.contacts), label=f"random pair {k}")
