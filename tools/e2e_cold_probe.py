"""Per-step e2e timings with and without the device tree cache (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_scene, scene_problems  # noqa: E402
from paper_2309_15417_b200 import ccd  # noqa: E402

sc = build_scene("c1", 0, None)
problems = scene_problems(sc)
pairs_obj = [pr[0][0] for pr in problems]
for cache in (True, False, True):
    ccd.set_tree_cache(cache)
    for i in range(6):
        torch.cuda.synchronize()
        tm = {}
        t0 = time.perf_counter()
        ccd.earliest_contacts(pairs_obj, sc.dt, timings=tm)
        t1 = time.perf_counter()
        print(cache, i, round(1e3 * (t1 - t0), 2), {k: round(v[0], 2) if k != "h2d_bytes" else v[0] for k, v in tm.items()},
              flush=True)
