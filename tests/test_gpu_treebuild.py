"""GPU surrogate-tree builder (ltsg_build_trees, treebuild.py) against the
reference: bit for bit on the reference-built fixtures of every BASELINE
mesh family (tests/golden/trees_gpu.npz), and at scene scale against the
host restatement plus the halo-cover invariant (surrogate.py:100-113)."""

import numpy as np
import pytest

from helpers import golden
from golden import scene_codec as SC

pytestmark = pytest.mark.gpu


def _same(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _assert_tree_equal(got, ref, what):
    assert got.level_sizes() == ref.level_sizes(), what
    for li, (a, b) in enumerate(zip(got.levels, ref.levels)):
        assert _same(a.corners, b.corners), (what, li, np.abs(np.asarray(a.corners) - b.corners).max())
        assert _same(a.epsilon, b.epsilon), (what, li)
        if b.children is None:
            assert a.children is None
        else:
            assert len(a.children) == len(b.children)
            for x, y in zip(a.children, b.children):
                assert np.array_equal(np.asarray(x), np.asarray(y)), (what, li)


def _cases():
    return golden("trees_gpu")["cases"]


def test_batched_build_matches_reference_trees():
    from paper_2309_15417_b200 import treebuild

    cases = [c for c in _cases() if int(c["fanout"]) == 4 and int(c["max_levels"]) == 8]
    trees = treebuild.build_surrogate_trees([c["corners"] for c in cases], [c["epsilon"] for c in cases])
    for c, t in zip(cases, trees):
        _assert_tree_equal(t, SC.decode_tree(c["tree"]), c["name"])


@pytest.mark.parametrize("name", ["fanout_2", "fanout_3", "fanout_8", "max_levels_3", "tie_plane", "c2_domino"])
def test_single_build_with_reference_parameters(name):
    from paper_2309_15417_b200 import treebuild

    c = next(c for c in _cases() if c["name"] == name)
    t = treebuild.build_surrogate_tree(c["corners"], c["epsilon"], fanout=int(c["fanout"]),
                                       max_levels=int(c["max_levels"]))
    _assert_tree_equal(t, SC.decode_tree(c["tree"]), name)


def test_reference_errors():
    from paper_2309_15417_b200 import treebuild

    c = _cases()[0]["corners"]
    with pytest.raises(ValueError):
        treebuild.build_surrogate_tree(c, 0.0)
    with pytest.raises(ValueError):
        treebuild.build_surrogate_tree(c, 0.01, fanout=1)
    with pytest.raises(ValueError):
        treebuild.build_surrogate_tree(c, 0.01, fanout=9)
    with pytest.raises(ValueError):
        treebuild.build_surrogate_tree(np.zeros((0, 3, 3)), 0.01)


def test_single_triangle_and_mesh_objects():
    from paper_2309_15417_b200 import treebuild

    tri = np.array([[[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]])
    t = treebuild.build_surrogate_tree(tri, 0.01)
    assert t.level_sizes() == [1] and t.levels[0].children is None

    class Mesh:  # the reference's TriangleMesh surface: corners() -> (a, b, c)
        def __init__(self, c):
            self.c = c

        def corners(self):
            return self.c[:, 0], self.c[:, 1], self.c[:, 2]

    c = next(c for c in _cases() if c["name"] == "c3_rock_0")
    t = treebuild.build_surrogate_tree(Mesh(c["corners"]), c["epsilon"])
    _assert_tree_equal(t, SC.decode_tree(c["tree"]), "mesh object")


def _blas_core():
    try:
        import ctypes
        import glob
        import os

        lib = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(np.__file__) + ".libs",
                                                 "libscipy_openblas64_*.so"))[0])
        f = lib.scipy_openblas_get_corename64_
        f.restype = ctypes.c_char_p
        return f().decode()
    except Exception:
        return "unknown"


def test_scene_scale_against_host_builder_and_cover_invariant():
    """c1/c4-shaped batch (512 noisy 1280-tri icospheres) plus c3 rocks and c5
    icospheres: every level equals the host numpy restatement when this host's
    OpenBLAS runs the kernels lapack3.cuh models, and on any host every parent
    covers its children's halos (surrogate.py:100-113)."""
    from oracle import tree_oracle as surrogate
    from paper_2309_15417_b200 import scenes, treebuild

    rng = np.random.default_rng(11)
    meshes, eps = [], []
    v0, f0 = scenes.icosphere(3)
    for _ in range(512):
        v = v0 * (1.0 + rng.uniform(-0.05, 0.05, size=len(v0)))[:, None]
        meshes.append(np.stack([v[f0[:, 0]], v[f0[:, 1]], v[f0[:, 2]]], axis=1))
        eps.append(0.01)
    for _ in range(64):
        v, f = scenes.rock(rng)
        v = v * float(np.exp(rng.uniform(np.log(0.5), np.log(5.0))))
        meshes.append(np.stack([v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]], axis=1))
        eps.append(0.005)
    for sub in (0, 1, 2, 4, 5):
        v, f = scenes.icosphere(sub)
        v = v * float(np.exp(rng.uniform(np.log(0.05), np.log(5.0))))
        meshes.append(np.stack([v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]], axis=1))
        eps.append(1e-3)
    trees = treebuild.build_surrogate_trees(meshes, eps)
    exact = _blas_core() == "SkylakeX"
    check = list(range(0, 512, 37)) + list(range(512, len(meshes)))
    for i in check:
        t = trees[i]
        if exact:
            _assert_tree_equal(t, surrogate.build_surrogate_tree(meshes[i], eps[i]), f"mesh {i}")
        for lvl in range(1, t.depth):
            par, fine = t.levels[lvl], t.levels[lvl - 1]
            for g, kids in enumerate(par.children):
                pts = fine.corners[kids].reshape(-1, 3)
                a, b, c = par.corners[g]
                d = surrogate._point_triangle_dist(pts, np.broadcast_to(a, pts.shape), np.broadcast_to(b, pts.shape),
                                                   np.broadcast_to(c, pts.shape))
                assert par.epsilon[g] >= (d + np.repeat(fine.epsilon[kids], 3)).max(), (i, lvl, g)
            # children partition the finer level
            allk = np.sort(np.concatenate(list(par.children)))
            assert np.array_equal(allk, np.arange(fine.size))
