"""CPU pins for the surrogate-tree builder.

* The reference-built fixtures (tests/golden/trees_gpu.npz, made by
  make_golden_trees.py from ltsdem.surrogate.build_surrogate_tree) equal
  the CPU tree oracle (oracle/tree_oracle.py) bit for bit on this host.
* The oracle's LAPACK restatement (oracle/lapack_svd.py, the algorithm
  csrc/lapack3.cuh implements) gives numpy's V^T bit for bit on every
  plane-fit group of the fixtures and on degenerate matrices.
* The device builder's level layout (treebuild.TreeLayout) matches the
  reference's level sizes.
"""

import numpy as np
import pytest

from helpers import golden
from golden import scene_codec as SC
from oracle import lapack_svd as L
from oracle import tree_oracle as S
from paper_2309_15417_b200.treebuild import TreeLayout, level_sizes


def _cases():
    return golden("trees_gpu")["cases"]


def _same(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_fixture_covers_the_baseline_families():
    names = {c["name"] for c in _cases()}
    for want in ("c1_noisy_icosphere_0", "c2_domino", "c3_rock_0", "c5_icosphere_5", "c5_box_0", "tie_cube",
                 "tie_plane", "flat_grid", "fanout_2", "fanout_8", "max_levels_3"):
        assert want in names


@pytest.mark.parametrize("name", ["c1_noisy_icosphere_0", "c2_domino", "c3_rock_0", "c3_rock_1", "c5_icosphere_2",
                                  "c5_box_0", "tie_cube", "tie_plane", "flat_grid", "fanout_2", "fanout_3",
                                  "fanout_8", "max_levels_3"])
def test_host_builder_matches_reference_fixture(name):
    case = next(c for c in _cases() if c["name"] == name)
    ref = SC.decode_tree(case["tree"])
    got = S.build_surrogate_tree(case["corners"], case["epsilon"], fanout=int(case["fanout"]),
                                 max_levels=int(case["max_levels"]))
    assert got.level_sizes() == ref.level_sizes()
    for a, b in zip(got.levels, ref.levels):
        assert _same(a.corners, b.corners) and _same(a.epsilon, b.epsilon)
        if b.children is not None:
            assert [list(x) for x in a.children] == [list(x) for x in b.children]


def _groups(case, limit_levels=3):
    """The plane-fit inputs `rel` of the first coarse levels of a fixture tree."""
    ref = SC.decode_tree(case["tree"])
    fan = int(case["fanout"])
    out = []
    for lvl in range(1, min(len(ref.levels), limit_levels + 1)):
        fine = ref.levels[lvl - 1].corners
        order = S.morton_order(S._row_mean(fine, 1))
        for g in range(0, len(order), fan):
            pts = fine[order[g:g + fan]].reshape(-1, 3)
            out.append(pts - S._row_mean(pts[None], 1)[0])
    return out


@pytest.mark.parametrize("name", ["c2_domino", "c3_rock_0", "c5_icosphere_1", "c5_box_1", "tie_cube", "tie_plane",
                                  "flat_grid", "fanout_2", "fanout_3", "fanout_8"])
def test_oracle_svd_matches_numpy_on_tree_groups(name):
    case = next(c for c in _cases() if c["name"] == name)
    groups = _groups(case)[:120]
    for rel in groups:
        vt = np.linalg.svd(rel, full_matrices=False)[2]
        _, mine = L.svd_vt(rel)
        assert _same(vt, mine), rel


def test_oracle_svd_matches_numpy_on_degenerate_matrices():
    rng = np.random.default_rng(2)
    for _ in range(150):
        a, b = rng.choice([0.5, 1.0, 0.25, 2.0], 2)
        cand = np.array([[a, 0, 0], [-a, 0, 0], [0, a, 0], [0, -a, 0], [0, 0, b], [0, 0, -b], [a, a, 0],
                         [-a, -a, 0], [a, -a, 0], [-a, a, 0], [0, 0, 0], [a, a, b], [-a, -a, -b]])
        m = int(rng.choice([3, 6, 9, 12]))
        pts = cand[rng.choice(len(cand), m)][:, rng.permutation(3)] * rng.choice([-1, 1], 3)
        rel = pts - pts.mean(axis=0)
        assert _same(np.linalg.svd(rel, full_matrices=False)[2], L.svd_vt(rel)[1]), rel


def test_oracle_dnrm2_is_the_x87_kernel():
    # known values: the correctly rounded norm differs from the x87 result
    # only at double-rounding ties; these checks pin the accumulator order
    assert L.dnrm2([3.0, 4.0]) == 5.0
    assert L.dnrm2([1e-200, 1e-200]) > 0.0  # x87 squares do not underflow
    rng = np.random.default_rng(5)
    for _ in range(200):
        x = rng.normal(size=int(rng.integers(2, 12)))
        assert abs(L.dnrm2(list(x)) - np.sqrt(np.sum(x * x))) <= 4.5e-16 * np.sqrt(np.sum(x * x))


def test_layout_level_sizes_match_reference_trees():
    cases = _cases()
    for c in cases:
        ref = SC.decode_tree(c["tree"])
        assert level_sizes(len(c["corners"]), int(c["fanout"]), int(c["max_levels"])) == ref.level_sizes()
    four = [c for c in cases if int(c["fanout"]) == 4 and int(c["max_levels"]) == 8]
    lay = TreeLayout([len(c["corners"]) for c in four], 4, 8)
    assert lay.n_records == sum(sum(SC.decode_tree(c["tree"]).level_sizes()) for c in four)
    # step rows: grouped by level, prefix sums per level, finer level feeds the coarse one
    for lvl in range(lay.n_levels):
        rows = lay.steps[lay.level_steps[lvl]:lay.level_steps[lvl + 1]]
        assert np.array_equal(rows[:, 4], np.concatenate([[0], np.cumsum(rows[:-1, 1])]))
        assert np.array_equal(rows[:, 5], np.concatenate([[0], np.cumsum(rows[:-1, 3])]))
        assert lay.level_keys[lvl] == rows[:, 1].sum() and lay.level_groups[lvl] == rows[:, 3].sum()
        assert np.all(rows[:, 3] == -(-rows[:, 1] // 4))
        assert np.all(rows[:, 2] == rows[:, 0] + rows[:, 1])
