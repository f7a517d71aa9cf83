import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2309_15417_b200 import broadphase as BP
from test_gpu_broadphase import _random_records
import torch
for n, side in ((2000, 30.0), (20000, 90.0), (200000, 200.0)):
    rng = np.random.default_rng(1)
    rec, srec = _random_records(rng, n, 1, side=side)
    pol = BP.TimeStepPolicy(dt_max=0.1)
    for _ in range(3): ga = BP.graph_arrays(rec, srec, pol)
    ms = []
    for _ in range(10):
        ga = BP.graph_arrays(rec, srec, pol); ms.append(ga.ms)
    t = time.perf_counter()
    for _ in range(10): BP.graph_arrays(rec, srec, pol)
    wall = (time.perf_counter() - t) / 10 * 1e3
    print(n, "edges", len(ga.edge), "links", len(ga.link), "cand", ga.candidates, "device ms", np.median(ms), "wall ms", wall, "launches", ga.launches)
