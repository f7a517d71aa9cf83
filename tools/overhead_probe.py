"""Host overhead of run_scene: wall time per call vs the library's device time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_scene, scene_problems  # noqa: E402
from paper_2309_15417_b200 import ccd, packing  # noqa: E402

for cfg in ("c2", "c1"):
    sc = build_scene(cfg, 0, None)
    ds = ccd.DeviceScene(packing.pack(scene_problems(sc)))
    for _ in range(3):
        ccd.run_scene(ds)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    n = 10
    for _ in range(n):
        r = ccd.run_scene(ds)
    ev1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e3
    print(cfg, "wall ms/call %.3f" % wall, "event ms/call %.3f" % (ev0.elapsed_time(ev1) / n), flush=True)
