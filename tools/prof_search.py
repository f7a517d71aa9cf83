"""One warm search of a config inside an NVTX range "prof" (for
`ncu --nvtx --nvtx-include prof/`): two untimed calls first (the first runs
the traversal in sync mode), then the profiled call, which runs async
(generation g is the g-th launch of each per-generation kernel)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2309_15417_b200 import ccd, packing, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--pairs", type=int, default=None)
ap.add_argument("--exhaustive", action="store_true")
a = ap.parse_args()
key = {"c1": "n_pairs", "c2": "n_boxes", "c3": "n_rocks", "c4": "n_pairs", "c5": "n_particles"}[a.config]
sc = scenes.CONFIGS[a.config](**({key: a.pairs} if a.pairs else {}))
from bench import scene_problems  # noqa: E402

import torch  # noqa: E402

ds = ccd.DeviceScene(packing.pack(scene_problems(sc)))
for _ in range(2):
    ccd.run_scene(ds, exhaustive=a.exhaustive)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
r = ccd.run_scene(ds, exhaustive=a.exhaustive)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("stats", r.stats)
