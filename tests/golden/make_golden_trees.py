"""Surrogate-tree fixtures for the GPU tree builder, made by running the
REFERENCE's `ltsdem.surrogate.build_surrogate_tree` (surrogate.py:71-119).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_trees.py

Output (committed): trees_gpu.npz -- the mesh families of every BASELINE
config, recentred the way make_particle does it (body.py:70-72), plus
degenerate meshes and non-default fanout / level caps:
  c1/c4   noisy 1280-tri icospheres (radial noise U(-0.05, 0.05))
  c2      the 0.1 x 0.5 x 1 domino box (12 tris, axis-aligned: exact zeros)
  c3      rocks (hull of 64 directions), radius log-uniform in [0.5, 5]
  c5      icospheres at 0..5 subdivisions (20...20480 tris) and 12-tri boxes,
          radius log-uniform in [0.05, 5] (size ratio 100:1)
  ties    the unit cube (equal singular values), the reference's make_plane
          and a flat 128-tri grid (a zero singular value, exact zeros)
  params  fanout 2, 3, 8 and max_levels 3 on a 320-tri sphere
The trees are stored with SC.encode_tree; each case keeps the level-0
corners, epsilon, fanout and max_levels it was built with.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from ltsdem.mesh import make_plane  # noqa: E402
from ltsdem.surrogate import build_surrogate_tree  # noqa: E402

import gio  # noqa: E402
import scene_codec as SC  # noqa: E402
from paper_2309_15417_b200 import bodies as B  # noqa: E402
from paper_2309_15417_b200 import scenes as S  # noqa: E402


def _centred_corners(v, f):
    v = np.asarray(v, dtype=np.float64)
    f = np.asarray(f, dtype=np.int64)
    c = v - B.centre_of_mass(v, f)
    return np.ascontiguousarray(np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1))


def main():
    rng = np.random.default_rng(230915417 + 77)
    cases = []

    def add(name, corners, eps, fanout=4, max_levels=8):
        t = build_surrogate_tree(corners, eps, fanout=fanout, max_levels=max_levels)
        cases.append({"name": name, "corners": corners, "epsilon": float(eps), "fanout": fanout,
                      "max_levels": max_levels, "tree": SC.encode_tree(t)})
        print(f"{name}: {t.level_sizes()}", flush=True)

    v0, f0 = S.icosphere(3)
    for k in range(2):
        v = v0 * (1.0 + rng.uniform(-0.05, 0.05, size=len(v0)))[:, None]
        add(f"c1_noisy_icosphere_{k}", _centred_corners(v, f0), 0.01)
    v, f = S.box((0.1, 0.5, 1.0))
    add("c2_domino", _centred_corners(v, f), 1e-3)
    for k in range(3):
        v, f = S.rock(rng)
        r = float(np.exp(rng.uniform(np.log(0.5), np.log(5.0))))
        add(f"c3_rock_{k}", _centred_corners(v * r, f), 0.005)
    for sub in range(6):
        v, f = S.icosphere(sub)
        r = float(np.exp(rng.uniform(np.log(0.05), np.log(5.0))))
        add(f"c5_icosphere_{sub}", _centred_corners(v * r, f), 1e-3)
    for k in range(2):
        v, f = S.box((1.0, 0.8, 0.6))
        r = float(np.exp(rng.uniform(np.log(0.05), np.log(5.0))))
        add(f"c5_box_{k}", _centred_corners(v * r, f), 1e-3)
    v, f = S.box((1.0, 1.0, 1.0))
    add("tie_cube", _centred_corners(v, f), 1e-3)
    plane = make_plane(np.array([-1.0, -1.0, 0.5]), np.array([1.0, 1.0, 0.5]))
    add("tie_plane", np.ascontiguousarray(np.stack(plane.corners(), axis=1)), 1e-3)
    g = np.linspace(-1.0, 1.0, 9)
    gx, gy = np.meshgrid(g, g, indexing="ij")
    gv = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)], axis=1)
    quads = [(i * 9 + j, (i + 1) * 9 + j, (i + 1) * 9 + j + 1, i * 9 + j + 1) for i in range(8) for j in range(8)]
    gf = np.array([t for a, b, c, d in quads for t in ((a, b, c), (a, c, d))], dtype=np.int64)
    add("flat_grid", np.ascontiguousarray(np.stack([gv[gf[:, 0]], gv[gf[:, 1]], gv[gf[:, 2]]], axis=1)), 1e-3)
    v, f = S.icosphere(2)
    v = v * (1.0 + rng.uniform(-0.05, 0.05, size=len(v)))[:, None]
    c = _centred_corners(v, f)
    for fanout in (2, 3, 8):
        add(f"fanout_{fanout}", c, 0.01, fanout=fanout)
    add("max_levels_3", c, 0.01, max_levels=3)
    gio.save(os.path.join(HERE, "trees_gpu.npz"), {"cases": cases})


if __name__ == "__main__":
    main()
