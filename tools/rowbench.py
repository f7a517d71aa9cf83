"""Microbenchmark: ltsg_feature_distances rows/s on mesh-derived rows.

mode "far": random triangle pairs of two spheres 2.0 apart (mostly far);
mode "near": pairs whose centroids are within 0.25 (the rows that survive
the traversal's sphere cull)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15417_b200 import _lib, scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
mode = sys.argv[2] if len(sys.argv) > 2 else "near"
rng = np.random.default_rng(0)
v, f = scenes.icosphere(3)
va = v * (1 + rng.uniform(-0.05, 0.05, len(v)))[:, None]
vb = v * (1 + rng.uniform(-0.05, 0.05, len(v)))[:, None] + np.array([2.0, 0.0, 0.0])
ca = np.stack([va[f[:, 0]], va[f[:, 1]], va[f[:, 2]]], 1)
cb = np.stack([vb[f[:, 0]], vb[f[:, 1]], vb[f[:, 2]]], 1)
if mode == "near":
    ma, mb = ca.mean(1), cb.mean(1)
    d = np.linalg.norm(ma[:, None, :] - mb[None, :, :], axis=2)
    ii, jj = np.nonzero(d < 0.25)
    pick = rng.integers(0, len(ii), n)
    ia, ib = ii[pick], jj[pick]
else:
    ia = rng.integers(0, len(f), n)
    ib = rng.integers(0, len(f), n)
ta = torch.from_numpy(np.ascontiguousarray(ca[ia])).cuda()
tb = torch.from_numpy(np.ascontiguousarray(cb[ib])).cuda()
d = torch.empty(n, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
L = _lib.lib()
for _ in range(3):
    L.ltsg_feature_distances(C.c_void_p(ta.data_ptr()), C.c_void_p(tb.data_ptr()), n, C.c_void_p(d.data_ptr()), st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    L.ltsg_feature_distances(C.c_void_p(ta.data_ptr()), C.c_void_p(tb.data_ptr()), n, C.c_void_p(d.data_ptr()), st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
tf = C.c_double()
pm = C.c_double()
L.ltsg_fp64_peak(C.byref(tf), C.byref(pm), st)
print(json.dumps({"lib": os.path.basename(os.environ.get("LTSG_LIB", "default")), "mode": mode, "rows": n, "ms": round(ms, 4),
                  "rows_per_s": n / ms * 1e3, "tflops_984": n * 984 / ms / 1e9, "frac": n * 984 / ms / 1e9 / tf.value,
                  "checksum": float(d.sum())}))
