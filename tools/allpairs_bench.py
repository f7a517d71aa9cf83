"""Microbenchmark of the exhaustive fine x fine distance kernels on c1 pairs:
the register x broadcast tile kernel (default) and the per-row staged kernel
(LTSG_ALLPAIRS_STAGED=1).  Prints rows/s and the fraction of the in-run FP64
peak at 984 flops per row."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15417_b200 import _lib, ccd, packing, scenes  # noqa: E402

n_pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tile", "staged"]
sc = scenes.config1(n_pairs=n_pairs)
ds = ccd.DeviceScene(packing.pack([([(sc.body(a), sc.body(b))], 0.0, 0.0) for a, b in sc.pairs]))
s = ds.struct(1e-3, False)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
L = _lib.lib()
tf, pm = C.c_double(), C.c_double()
_lib.check(L.ltsg_fp64_peak(C.byref(tf), C.byref(pm), st), "peak")
for v in variants:
    if v == "staged":
        os.environ["LTSG_ALLPAIRS_STAGED"] = "1"
    else:
        os.environ.pop("LTSG_ALLPAIRS_STAGED", None)
    best = None
    for _ in range(4):
        rows, hits, ms = C.c_int64(), C.c_int64(), C.c_double()
        _lib.check(L.ltsg_exhaustive_rows(C.byref(s), C.byref(rows), C.byref(hits), C.byref(ms),
                                          _lib.workspace().handle, st), "rows")
        best = ms.value if best is None else min(best, ms.value)
    tfl = rows.value * 984 / (best * 1e-3) / 1e12
    print(json.dumps({"variant": v, "pairs": n_pairs, "rows": rows.value, "hits": hits.value, "ms": round(best, 4),
                      "rows_per_s": rows.value / best * 1e3, "tflops": round(tfl, 3),
                      "frac": round(tfl / tf.value, 4), "peak": round(tf.value, 2)}))
