"""Phase trace of one warm search (LTSG_TRACE=1 on the last call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse

from paper_2309_15417_b200 import ccd, packing, scenes

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--pairs", type=int, default=None)
a = ap.parse_args()
kw = {"n_pairs": a.pairs} if a.pairs else {}
sc = scenes.CONFIGS[a.config](**kw)
from bench import scene_problems  # noqa: E402

hs = packing.pack(scene_problems(sc))
import torch
ds = ccd.DeviceScene(hs)
for _ in range(4):
    ccd.run_scene(ds)
torch.cuda.synchronize()
os.environ["LTSG_TRACE"] = "1"
r = ccd.run_scene(ds)
torch.cuda.synchronize()
print("problems", len(r), "stats", r.stats)
