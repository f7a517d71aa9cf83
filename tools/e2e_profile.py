"""Profile the e2e path of bench.py (host bodies -> results) with cProfile."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_15417_b200 import ccd, packing, scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
sc = scenes.config1(n_pairs=n)
pairs = [(sc.body(a), sc.body(b)) for a, b in sc.pairs]
problems = [([p], 0.0, 0.0) for p in pairs]
ds = ccd.DeviceScene(packing.pack(problems))
for _ in range(3):
    ccd.run_scene(ds)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(5):
    flush.fill_(1)
    torch.cuda.synchronize()
    tm = {}
    t0 = time.perf_counter()
    if it == 4:
        pr = cProfile.Profile()
        pr.enable()
    out = ccd.earliest_contacts(pairs, sc.dt, timings=tm)
    if it == 4:
        pr.disable()
    t1 = time.perf_counter()
    print(it, round(1e3 * (t1 - t0), 2), {k: round(v[0], 2) for k, v in tm.items()})
pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
