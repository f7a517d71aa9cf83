"""GPU parity of the exhaustive fine x fine distance kernel (k_allpairs_tile,
the roofline kernel): every row's ccd._feature_distances value (ccd.py:135-153)
bit for bit against the CPU oracle, and the hit count of ltsg_exhaustive_rows
against the oracle's count of rows within h + 1e-9 (ccd.py:407)."""

import ctypes as C

import numpy as np
import pytest

from oracle import narrow_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_15417_b200 import _lib, ccd, packing

    return torch, _lib, ccd, packing


def _oracle_rows(hs, pairs):
    """Oracle distances of every fine row, in the kernel's output order."""
    slot = {}
    for a, b in pairs:  # body slots in first-appearance order (packing._tables)
        for x in (a, b):
            slot.setdefault(id(x), len(slot))
    out = []
    for a, b in pairs:
        ra, rb = O.RigidPath(a), O.RigidPath(b)
        na, nb = a.tree.levels[0].size, b.tree.levels[0].size
        oa = hs.tri_orig[hs.body_levels[slot[id(a)], 2]:][:na]
        ob = hs.tri_orig[hs.body_levels[slot[id(b)], 2]:][:nb]
        wa = ra.world(0, oa, np.zeros(na))
        wb = rb.world(0, ob, np.zeros(nb))
        ia, ib = np.repeat(np.arange(na), nb), np.tile(np.arange(nb), na)
        out.append(O.tri_pair_distance(wa[ia], wb[ib]))
    return np.concatenate(out)


def _run(env, pairs):
    torch, _lib, ccd, packing = env
    hs = packing.pack([([p], 0.0, 0.0) for p in pairs])
    ds = ccd.DeviceScene(hs)
    sc = ds.struct(1e-3, False)
    n = sum(a.tree.levels[0].size * b.tree.levels[0].size for a, b in pairs)
    dist = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    rows = C.c_int64()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.lib().ltsg_exhaustive_distances(C.byref(sc), C.c_void_p(dist.data_ptr()), C.byref(rows),
                                                    _lib.workspace().handle, st), "ltsg_exhaustive_distances")
    r2, hits, ms = C.c_int64(), C.c_int64(), C.c_double()
    _lib.check(_lib.lib().ltsg_exhaustive_rows(C.byref(sc), C.byref(r2), C.byref(hits), C.byref(ms),
                                               _lib.workspace().handle, st), "ltsg_exhaustive_rows")
    torch.cuda.synchronize()
    assert rows.value == n and r2.value == n
    return hs, dist.cpu().numpy(), hits.value


def _check(env, pairs):
    hs, got, hits = _run(env, pairs)
    want = _oracle_rows(hs, pairs)
    bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
    assert len(bad) == 0, f"{len(bad)} of {len(want)} rows differ, first {bad[:5]}: {got[bad[:5]]} vs {want[bad[:5]]}"
    h = np.concatenate([np.full(a.tree.levels[0].size * b.tree.levels[0].size,
                                a.tree.levels[0].epsilon[0] + b.tree.levels[0].epsilon[0]) for a, b in pairs])
    assert hits == int(np.count_nonzero(want <= h + 1e-9))


def test_allpairs_c1_rows_bit_exact(env):
    from paper_2309_15417_b200 import scenes

    sc = scenes.config1(n_pairs=3, subdiv=2)
    _check(env, [(sc.body(a), sc.body(b)) for a, b in sc.pairs])


def test_allpairs_ragged_tiles_and_mixed_sizes(env):
    """Pairs whose sizes are not multiples of the tile edges (boxes, rocks,
    icospheres of different depth), both body orders."""
    from paper_2309_15417_b200 import scenes

    s3 = scenes.config3(n_rocks=12)
    rocks = list(s3.particles.values())
    s1 = scenes.config1(n_pairs=2, subdiv=1)
    ico = list(s1.particles.values())
    s2 = scenes.config2(n_boxes=4)
    boxes = list(s2.particles.values())
    pairs = [(rocks[0], rocks[1]), (ico[0], rocks[2]), (rocks[3], ico[1]), (boxes[0], boxes[1]),
             (boxes[2], ico[2]), (rocks[4], boxes[3])]
    _check(env, pairs)


def _degenerate_rows(rng):
    """Triangle pairs that leave the distance kernel's fast paths: repeated
    and collinear corners, tiny and huge scales (|e|^2 outside the regular
    range), parallel and collinear edges, coplanar, identical and touching
    triangles, exact zeros."""
    base = rng.normal(size=(64, 3, 3))
    other = rng.normal(size=(64, 3, 3)) * 0.5
    rows_a, rows_b = [], []
    dup = base.copy()
    dup[:, 1] = dup[:, 0]
    col = base.copy()
    col[:, 2] = col[:, 0] + rng.uniform(-2, 2, (64, 1)) * (col[:, 1] - col[:, 0])
    for ta in (dup, col):
        rows_a.append(ta)
        rows_b.append(other + ta.mean(1, keepdims=True))
    for s in (1e-160, 1e-80, 1e-45, 1e40, 1e60):  # |e|^2 around and beyond 2^-150 .. 2^150
        rows_a.append(base * s)
        rows_b.append((base[:, [1, 2, 0]] + other * 0.1) * s)
    par_a = base.copy()
    par_b = base + rng.normal(size=(64, 1, 3)) * 0.3  # translated copy: every edge parallel
    rows_a += [par_a, base, base]
    rows_b += [par_b, base.copy(), base[:, [2, 0, 1]]]  # identical triangles (d = 0), permuted
    touch = base.copy()
    touch_b = rng.normal(size=(64, 3, 3))
    touch_b[:, 0] = touch[:, 1]  # shared vertex
    flat_a = base.copy()
    flat_a[:, :, 2] = 0.0
    flat_b = rng.normal(size=(64, 3, 3)) * 0.7
    flat_b[:, :, 2] = 0.0  # coplanar
    rows_a += [touch, flat_a]
    rows_b += [touch_b, flat_b]
    small_int = rng.integers(-3, 4, size=(64, 3, 3)).astype(float)  # exact zeros and ties
    rows_a.append(small_int)
    rows_b.append(rng.integers(-3, 4, size=(64, 3, 3)).astype(float))
    return np.concatenate(rows_a), np.concatenate(rows_b)


def test_row_distances_degenerate_bit_exact(env):
    """ltsg_feature_distances (the tile kernels' distance code) on rows that
    take the irregular-triangle and division fallbacks, bit for bit."""
    from paper_2309_15417_b200 import kernels

    ta, tb = _degenerate_rows(np.random.default_rng(7))
    got = kernels.feature_distances(ta, tb)
    want = O.tri_pair_distance(ta, tb)
    bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
    assert len(bad) == 0, f"{len(bad)} rows differ, first {bad[:5]}: {got[bad[:5]]} vs {want[bad[:5]]}"
