"""Time the device tree builder against the host numpy builder on the c1
mesh family (noisy 1280-tri icospheres), and check they agree."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import tree_oracle as surrogate  # noqa: E402
from paper_2309_15417_b200 import scenes, treebuild  # noqa: E402


def main(n=2048):
    import torch

    rng = np.random.default_rng(1)
    v0, f0 = scenes.icosphere(3)
    C = []
    for _ in range(n):
        v = v0 * (1.0 + rng.uniform(-0.05, 0.05, size=len(v0)))[:, None]
        C.append(np.stack([v[f0[:, 0]], v[f0[:, 1]], v[f0[:, 2]]], axis=1))
    treebuild.build_surrogate_trees(C[:8], [0.01] * 8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    trees = treebuild.build_surrogate_trees(C, [0.01] * n)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = surrogate.build_surrogate_trees(np.stack(C[:256]), 0.01)
    t_host = (time.perf_counter() - t0) * n / 256
    same = all(np.array_equal(a.corners.view(np.uint64), b.corners.view(np.uint64)) and
               np.array_equal(a.epsilon.view(np.uint64), b.epsilon.view(np.uint64))
               for ta, tb in zip(trees[:256], host) for a, b in zip(ta.levels, tb.levels))
    print(f"{n} trees of 1280 tris: gpu {t_gpu * 1e3:.1f} ms (incl. H2D/D2H and tree objects), "
          f"host numpy (vectorised, 1 core) {t_host * 1e3:.0f} ms extrapolated; identical: {same}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2048)
