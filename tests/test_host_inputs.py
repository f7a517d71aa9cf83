"""Host-side input construction and packing (no GPU)."""

import numpy as np
import pytest

from helpers import golden
from golden import scene_codec as SC
from paper_2309_15417_b200 import bodies as B
from paper_2309_15417_b200 import packing, scenes
from oracle.tree_oracle import build_surrogate_tree


@pytest.mark.parametrize("k", range(8))
def test_tree_builder_matches_reference_trees(k):
    case = golden("trees")["trees"][k]
    v, f = case["vertices"], case["triangles"]
    ref = SC.decode_tree(case["tree"])
    corners = np.stack([v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]], axis=1)
    got = build_surrogate_tree(corners, case["epsilon"])
    assert got.level_sizes() == ref.level_sizes()
    for a, b in zip(got.levels, ref.levels):
        # bit-exact on the build host; LAPACK may differ in the last bits elsewhere
        np.testing.assert_allclose(a.corners, b.corners, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(a.epsilon, b.epsilon, rtol=1e-12, atol=1e-14)
        if b.children is not None:
            for ca, cb in zip(a.children, b.children):
                np.testing.assert_array_equal(ca, cb)


def test_icosphere_counts():
    for s in range(4):
        v, f = scenes.icosphere(s)
        assert len(f) == 20 * 4 ** s
        assert len(v) == 10 * 4 ** s + 2
        np.testing.assert_allclose(np.linalg.norm(v, axis=1), 1.0)


def _tree_of(n_sub=2):
    v, f = scenes.icosphere(n_sub)
    return build_surrogate_tree(np.stack([v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]], 1), 0.01)


def test_packed_children_are_contiguous_and_map_back():
    tree = _tree_of(2)
    pt = packing._pack_tree(tree)
    L = len(tree.levels)
    for lvl in range(1, L):
        off, size = pt.level_off[lvl], pt.level_size[lvl]
        fine_off = pt.level_off[lvl - 1]
        for r in range(size):
            rec = pt.records[off + r]
            ch = rec[11:12].view(np.uint64)[0]
            first, count = int(ch & np.uint64(0xFFFFFFFF)), int(ch >> np.uint64(32))
            parent = pt.orig[off + r]
            want = sorted(tree.levels[lvl].children[parent])
            got = sorted(pt.orig[fine_off + first: fine_off + first + count])
            assert got == want
    for lvl in range(L):
        off, size = pt.level_off[lvl], pt.level_size[lvl]
        np.testing.assert_array_equal(pt.records[off:off + size, :9].reshape(-1, 3, 3),
                                      tree.levels[lvl].corners[pt.orig[off:off + size]])
        np.testing.assert_array_equal(pt.records[off:off + size, 9],
                                      tree.levels[lvl].epsilon[pt.orig[off:off + size]])


def test_pack_groups_and_shared_bodies():
    tree = _tree_of(1)
    a = B.Particle(0, tree, 0.01, 1.0, B.timeline(B.state((0, 0, 0))))
    b = B.Particle(1, tree, 0.01, 1.0, B.timeline(B.state((2, 0, 0))))
    c = B.Particle(2, tree, 0.01, 1.0, B.timeline(B.state((4, 0, 0))))
    s = B.StaticBody(-1, tree, 0.01)
    hs = packing.pack([([(a, b)], 0.0, 0.0), ([(b, c), (a, c), (c, s), (a, c)], 0.5, 1.0)])
    assert len(hs.body_state) == 4          # shared objects packed once
    assert hs.n_tris == sum(l.size for l in tree.levels)  # one tree copy
    assert len(hs.up_table) == 1
    assert hs.pair_problem.tolist() == [0, 1, 1, 1, 1]
    # groups rank the distinct (id_a, id_b) pairs of each problem
    assert hs.pair_group.tolist() == [0, 1, 0, 2, 0]
    assert hs.body_state[3, 13] == 1.0 and hs.body_levels[3, 1] == -1


def test_scenes_are_seeded():
    s1 = scenes.config1(n_pairs=3, subdiv=1)
    s2 = scenes.config1(n_pairs=3, subdiv=1)
    for k in s1.particles:
        np.testing.assert_array_equal(s1.particles[k].timeline.current.position,
                                      s2.particles[k].timeline.current.position)
        np.testing.assert_array_equal(s1.particles[k].tree.levels[0].corners,
                                      s2.particles[k].tree.levels[0].corners)


def test_domino_pairs_are_sphere_overlaps():
    s = scenes.config2(n_boxes=40)
    r = s.particles[0].radius
    assert abs(r - (np.sqrt(0.05 ** 2 + 0.25 ** 2 + 0.5 ** 2) + 1e-3)) < 1e-12
    assert all(0.18 * (b - a) <= 2 * r for a, b in s.pairs)
    assert len(s.pairs) == sum(min(6, 39 - i) for i in range(40))


def test_batched_particles_match_single_builds():
    from paper_2309_15417_b200.bodies import make_particle

    rng = np.random.default_rng(3)
    meshes = scenes._noisy_icosphere_trees(rng, 1030, 1, 0.05, 0.01)
    states = [B.state(np.zeros(3)) for _ in meshes]
    made = scenes.make_particles(range(1030), meshes, 0.01, states)
    for k in (0, 517, 1029):
        v, f = meshes[k]
        c = v - B.centre_of_mass(v, f)
        single = build_surrogate_tree(np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1), 0.01)
        ref = make_particle(k, v, f, 0.01, states[k], tree=single)
        assert made[k].radius == ref.radius
        for a, b in zip(made[k].tree.levels, ref.tree.levels):
            np.testing.assert_array_equal(a.corners, b.corners)
            np.testing.assert_array_equal(a.epsilon, b.epsilon)
            if b.children is not None:
                assert len(a.children) == len(b.children)
                for x, y in zip(a.children, b.children):
                    np.testing.assert_array_equal(x, y)


def _expand_upload(hs):
    """Host restatement of ltsg_unpack_trees for slots 0..11."""
    out = np.zeros((hs.n_tris, 12))
    for rec_off, n0, nc, vo, io, co, eo, mode in hs.up_table:
        vidx = hs.up_vidx[io:io + n0]
        out[rec_off:rec_off + n0, :9] = hs.up_verts[vo + vidx].reshape(n0, 9)
        out[rec_off + n0:rec_off + n0 + nc, :9] = hs.up_coarse[co:co + nc]
        if mode:
            out[rec_off:rec_off + n0 + nc, 9] = hs.up_eps[eo:eo + n0 + nc]
        else:
            out[rec_off:rec_off + n0, 9] = hs.up_eps[eo]
            out[rec_off + n0:rec_off + n0 + nc, 9] = hs.up_eps[eo + 1:eo + 1 + nc]
        kids = np.zeros((n0 + nc, 2), dtype=np.int32)
        kids[n0:] = hs.up_kids[co:co + nc]
        out[rec_off:rec_off + n0 + nc, 11] = kids.view(np.float64).reshape(-1)
    return out


def test_compact_upload_image_rebuilds_records():
    trees = [_tree_of(1), _tree_of(2)]
    bodies = [B.Particle(i, t, 0.01, 1.0, B.timeline(B.state((2.0 * i, 0, 0)))) for i, t in enumerate(trees)]
    hs = packing.pack([([(bodies[0], bodies[1])], 0.0, 0.0)])
    rec = hs.records()
    got = _expand_upload(hs)
    keep = [k for k in range(12) if k != 10]  # slot 10 (arm) is derived on the device
    assert got[:, keep].view(np.uint64).tolist() == rec[:, keep].view(np.uint64).tolist()
    # the fine level is shared-vertex compressed
    n0 = sum(int(pt.level_size[0]) for pt in hs.trees)
    assert len(hs.up_verts) < 3 * n0 / 2
    assert hs.nbytes < 0.6 * (rec.nbytes + hs.tri_orig.nbytes)


def test_compact_upload_keeps_signed_zero_apart():
    corners = np.array([[[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]],
                        [[-0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]]])
    tree = build_surrogate_tree(corners, 0.01)
    pt = packing._pack_tree(tree)
    rebuilt = pt.verts[pt.vidx].reshape(-1, 9)
    assert rebuilt.view(np.uint64).tolist() == pt.records[:2, :9].view(np.uint64).tolist()
