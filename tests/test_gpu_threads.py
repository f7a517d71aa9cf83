"""The public API called from an engine-style thread pool (the reference's
`engine.step` runs `_compute_cluster` on a ThreadPoolExecutor,
engine.py:183-193): every thread gets its own workspace, packer and result
buffers, and all of them draw device memory from one process-wide pool.
Results must equal the serial calls bit for bit."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from helpers import compare_contacts, golden, run_case
from golden import scene_codec as SC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_15417_b200 import ccd

    return ccd


def _same(a, b, label):
    assert a.dt == b.dt and a.collision == b.collision and a.first_contact == b.first_contact, label
    compare_contacts(SC.encode_contacts(a.contacts), SC.encode_contacts(b.contacts), label=label)


@pytest.mark.parametrize("threads", [4, 8])
def test_thread_pool_equals_serial(G, threads):
    cases = golden("scenes_configs")["cases"] + golden("scenes_ccd")["cases"] + golden("scenes_crit2")["cases"][:40]
    serial = [run_case(G, c) for c in cases]
    work = list(range(len(cases))) * 3
    np.random.default_rng(threads).shuffle(work)
    with ThreadPoolExecutor(max_workers=threads) as ex:
        got = list(ex.map(lambda i: (i, run_case(G, cases[i])), work))
    for i, res in got:
        _same(res, serial[i], cases[i]["name"])


def test_thread_pool_cluster_batches(G):
    """effective_dts (one launch over a sweep's clusters) from several
    threads at once, each on its own stream, equals the serial call."""
    import torch
    from types import SimpleNamespace

    from paper_2309_15417_b200 import scenes

    scene = scenes.config5(n_particles=60, max_subdiv=2)
    clusters, plist = [], []
    for p in range(scene.n_problems):
        sel = np.flatnonzero(scene.problem == p)
        clusters.append(SimpleNamespace(dt=scene.dt[p], t_current=scene.t_base[p]))
        plist.append([scene.pairs[i] for i in sel])
    serial, _ = G.effective_dts(clusters, scene.particles, scene.statics, plist)

    def job(k):
        with torch.cuda.stream(torch.cuda.Stream()):
            out, _ = G.effective_dts(clusters, scene.particles, scene.statics, plist)
        return out

    with ThreadPoolExecutor(max_workers=6) as ex:
        runs = list(ex.map(job, range(12)))
    for out in runs:
        for p, (a, b) in enumerate(zip(out, serial)):
            _same(a, b, f"cluster {p}")


def test_run_scene_on_a_side_stream(G):
    """run_scene(stream=s) orders the search after the scene upload on the
    current stream and reads the results back on `s`."""
    import torch

    from paper_2309_15417_b200 import packing

    case = golden("scenes_configs")["cases"][0]
    a, b = SC.decode_body(case["bodies"][0]), SC.decode_body(case["bodies"][1])
    hs = packing.pack([([(a, b)], case["dt"], 0.0)])
    ref = G.run_scene(G.DeviceScene(hs)).result(0)
    for _ in range(3):
        side = torch.cuda.Stream()
        got = G.run_scene(G.DeviceScene(hs), stream=side).result(0)
        _same(got, ref, "side stream")


def test_device_memory_pool_is_shared():
    """Workspaces of different threads draw from one pool: the capacity
    error class and the out-of-memory class are distinct."""
    from paper_2309_15417_b200 import _lib

    assert issubclass(_lib.CapacityError, _lib.LtsgError)
    assert issubclass(_lib.DeviceMemoryError, _lib.LtsgError)
    assert not issubclass(_lib.DeviceMemoryError, _lib.CapacityError)
