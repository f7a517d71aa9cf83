"""Benchmark of the B200 narrow phase.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1] [--pairs P]

One step = one batched narrow-phase pass (ltsg_search) over the whole
workload of the configuration: for c1, 1024 static pairs of 1280-triangle
noisy icospheres (BASELINE.json configs[0]).  Inputs are seeded synthetic
scenes (no dataset exists for this path).  Rank 0 prints ONE JSON line.

  value    reference-equivalent triangle-pair tests per second (the rows the
           reference's _feature_distances evaluates for the same search:
           screen + zoom + bisection), inputs resident in HBM, device time
  e2e      the same metric through the public batched API
           (`ccd.earliest_contacts`) from host bodies: packing, H2D copies,
           the search and the D2H copy of every result inside the timed region
  roofline the exact-distance kernel (k_screen_static for static batches,
           k_screen for moving ones): 984 FP64 flops per exact row over its
           CUDA-event time, against the FP64 DFMA peak measured in this run
  cpu_baseline  the CPU oracle (numpy restatement of the reference) on a
           bounded sample of the same workload, on this host's cores

`--impl reference` times the CPU oracle alone (the reference is pure
Python/numpy and cannot travel to the GPU box; the oracle is bit-identical
to it on the golden fixtures) and prints the same line with "impl".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FLOPS_PER_TEST = 984  # 6 x 62 point-triangle + 9 x 68 segment-segment
METRIC = "triangle-pair distance tests/sec"
CONFIG_DOC = {
    "c1": "1024 static pairs of 1280-tri noisy icospheres, centre distance U(1.9,2.1), eps 0.01, dt 0",
    "c2": "4096 domino boxes (12 tris), neighbour pairs within bounding-sphere overlap, eps 1e-3, dt 0",
    "c3": "20k convex rocks (~124 tris) packed at phi~0.55, bounding-sphere pairs, eps 0.005, dt 0",
    "c4": "8192 moving pairs of 1280-tri icospheres, v~N(0,1), w~N(0,2), gap U(0,0.5), eps 1e-3, dt 0.1",
    "c5": "2000 polydisperse mixed meshes, clusters of the swept-sphere graph, eps 1e-3, dt 0.1",
}


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def build_scene(config: str, rank: int, pairs: int | None):
    from paper_2309_15417_b200 import scenes

    fn = scenes.CONFIGS[config]
    kw = {"seed_offset": 100 * rank + int(config[1])}
    if pairs is not None:
        key = {"c1": "n_pairs", "c2": "n_boxes", "c3": "n_rocks", "c4": "n_pairs", "c5": "n_particles"}[config]
        kw[key] = pairs
    return fn(**kw)


def scene_problems(scene):
    """(pairs of body objects, dt, t_base) per problem, as the public API packs them."""
    import numpy as np

    if scene.mode == "pair":
        return [([(scene.body(a), scene.body(b))], float(scene.dt[k]), 0.0)
                for k, (a, b) in enumerate(scene.pairs)]
    probs = []
    for p in range(scene.n_problems):
        sel = np.flatnonzero(scene.problem == p)
        probs.append(([(scene.body(scene.pairs[i][0]), scene.body(scene.pairs[i][1])) for i in sel],
                      float(scene.dt[p]), float(scene.t_base[p])))
    return probs


def committed_traffic(config: str, kernel: str) -> dict:
    """DRAM bytes of the dominant kernel from the newest committed ncu summary
    (profiles/rNN_traffic_<config>.json, written by tools/traffic.py)."""
    import glob

    for path in sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_traffic_{config}.json")), reverse=True):
        try:
            d = json.load(open(path))
        except (OSError, ValueError):
            continue
        if d.get("kernel") == kernel:
            return d
    return {}


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU arms

def _oracle_job(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import narrow_oracle as O

    idx = args
    pairs, dt, tb = _CPU_PROBLEMS[idx]
    t0 = time.perf_counter()
    if len(pairs) == 1 and tb == 0.0:
        res = O.pair_earliest_contact(pairs[0][0], pairs[0][1], dt, exhaustive=_CPU_EXHAUSTIVE)
    else:
        from types import SimpleNamespace

        parts, stats, plist = {}, {}, []
        for a, b in pairs:
            for x in (a, b):
                (parts if hasattr(x, "timeline") else stats)[_bid(x)] = x
            plist.append((_bid(a), _bid(b)))
        res = O.compute_effective_dt(SimpleNamespace(dt=dt, t_current=tb), parts, stats, plist)
    rows = res.stats.get("rows", 0) + res.stats.get("zoom_rows", 0) + res.stats.get("bisect_rows", 0)
    return rows, len(res.raw), time.perf_counter() - t0


def _bid(b):
    return int(b.pid) if hasattr(b, "timeline") else int(b.sid)


_CPU_PROBLEMS = []
_CPU_EXHAUSTIVE = False


def cpu_sample(problems, n_items: int, workers: int, exhaustive: bool = False):
    """Run the oracle over the first n_items problems on `workers` processes."""
    import multiprocessing as mp

    global _CPU_PROBLEMS, _CPU_EXHAUSTIVE
    _CPU_PROBLEMS = problems
    _CPU_EXHAUSTIVE = exhaustive
    idx = list(range(min(n_items, len(problems))))
    t0 = time.perf_counter()
    if workers <= 1:
        out = [_oracle_job(i) for i in idx]
    else:
        with mp.get_context("fork").Pool(workers) as pool:
            out = pool.map(_oracle_job, idx, chunksize=1)
    wall = time.perf_counter() - t0
    rows = sum(o[0] for o in out)
    contacts = sum(o[1] for o in out)
    return rows, contacts, wall, len(idx)


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on this host's cores."""
    if rank != 0:
        return 0
    scene = build_scene(args.config, 0, args.pairs)
    problems = scene_problems(scene)
    workers = max(1, min(cpu_cores(), args.cpu_workers or cpu_cores()))
    per_step = max(workers, 1)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_sample(problems, min(per_step, 2), min(workers, 2))
    rows = contacts = 0
    wall = 0.0
    for s in range(args.steps):
        r, c, w, _ = cpu_sample(problems[s * per_step % max(len(problems), 1):] or problems,
                                per_step, workers)
        rows += r
        contacts += c
        wall += w
    value = rows / wall if wall > 0 else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tests/s",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": args.config, "description": CONFIG_DOC[args.config],
                   "sample_problems_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "tests/s", "cores": workers, "kind": "port",
                         "sample": f"{per_step} {args.config} problems per step x {args.steps} steps"},
        "e2e": {"value": value, "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "contacts_per_s": contacts / wall if wall > 0 else 0.0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import numpy as np
    import torch

    from paper_2309_15417_b200 import _lib, ccd, packing

    # host setup first: the scene builders fork worker processes, which must
    # happen before this process starts CUDA
    t_build = time.perf_counter()
    scene = build_scene(args.config, rank, args.pairs)
    problems = scene_problems(scene)
    hs = packing.pack(problems)
    t_build = time.perf_counter() - t_build

    # CPU baseline leg (rank 0 only): the oracle on this host's cores over a
    # bounded sample of the same workload, run before this process starts CUDA
    cpu = None
    if rank == 0 and not args.no_cpu:
        workers = max(1, min(cpu_cores(), 64))
        per_worker = 1 if args.exhaustive else 2  # an exhaustive c1 pair is ~40 s of numpy
        r, c, w, n = cpu_sample(problems, min(len(problems), per_worker * workers), workers, args.exhaustive)
        cpu = {"value": r / w if w > 0 else 0.0, "unit": "tests/s", "cores": workers, "kind": "port",
               "sample": f"{n} {args.config} problems (of {len(problems)}) through the numpy oracle, "
                         f"{workers} processes, {w:.1f} s wall"}

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    # The scene holds ~10^6 long-lived numpy objects (the reference's tree
    # format keeps one children array per surrogate triangle); exclude them
    # from cyclic GC scans, as a long-running engine would.
    import gc

    gc.collect()
    gc.freeze()
    ds = ccd.DeviceScene(hs)
    torch.cuda.synchronize()

    peak_tflops = C.c_double(0.0)
    peak_ms = C.c_double(0.0)
    _lib.check(_lib.lib().ltsg_fp64_peak(C.byref(peak_tflops), C.byref(peak_ms),
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "ltsg_fp64_peak")

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    # roofline of the 15-feature distance itself: every fine x fine row of a
    # sample of pairs evaluated exactly at tau = 0 (ltsg_exhaustive_rows)
    allpairs = None
    if scene.mode == "pair" and not args.no_allpairs:
        sub = problems[: min(len(problems), 16)]
        ds_sub = ccd.DeviceScene(packing.pack(sub))
        sc_sub = ds_sub.struct(1e-3, False)
        rows_c, hits_c, ms_c = C.c_int64(), C.c_int64(), C.c_double()
        for _ in range(2):
            _lib.check(_lib.lib().ltsg_exhaustive_rows(C.byref(sc_sub), C.byref(rows_c), C.byref(hits_c),
                                                       C.byref(ms_c), _lib.workspace().handle,
                                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                       "ltsg_exhaustive_rows")
        ach = rows_c.value * FLOPS_PER_TEST / (ms_c.value * 1e-3) / 1e12
        allpairs = {"kernel": "k_allpairs_tile", "pairs": len(sub), "rows": rows_c.value, "hits": hits_c.value,
                    "ms": ms_c.value, "tests_per_s": rows_c.value / (ms_c.value * 1e-3),
                    "achieved_tflops": ach, "frac": ach / peak_tflops.value}
        del ds_sub

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    # ---- device-resident steps
    for _ in range(args.warmup):
        res = ccd.run_scene(ds, exhaustive=args.exhaustive)
    stats = []
    step_ms = []
    barrier()
    # clocks and throttle reasons sampled across both timed loops (device, e2e)
    clocks = ClockSampler(local_rank).__enter__()
    for _ in range(args.steps):
        flush.fill_(1)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        res = ccd.run_scene(ds, exhaustive=args.exhaustive)
        ev1.record()
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        stats.append(res.stats)
    barrier()
    total_ms = sum(step_ms)
    tests = sum(s["rows_screen"] + s["rows_zoom"] + s["rows_bisect"] for s in stats)
    contacts = sum(s["n_raw"] for s in stats)
    # per-kernel device time of the screen from the library's own events
    screen_ms = sum(s.get("ms_screen", 0.0) for s in stats)
    screen_rows = sum(s["rows_screen"] for s in stats)
    exact_rows = sum(s.get("rows_screen_exact", s["rows_screen"]) for s in stats)
    exact_ms = sum(s.get("ms_exact", 0.0) for s in stats)
    expand_ms = sum(s.get("ms_expand", 0.0) for s in stats)
    launches = sum(s.get("launches", 0) for s in stats)

    # ---- end to end through the public API from host bodies.  Every step
    # packs the bodies' current states, copies the step's inputs H2D from
    # pinned memory, searches and reads the results back.  The surrogate
    # trees are immutable geometry: the public API keeps them
    # resident on the device after the first call (ccd.DeviceScene
    # cache_trees), so a step uploads the kinematic states and pair tables.
    # The same loop with the tree cache off (every step uploads the compact
    # geometry too) is reported as e2e_cold.
    pairs_obj = [pr[0][0] for pr in problems] if scene.mode == "pair" else None

    def e2e_loop(n_warm, n_timed):
        ms, ph = [], {}
        out = None
        for i in range(n_warm + n_timed):
            flush.fill_(1)
            torch.cuda.synchronize()
            tm = ph if i >= n_warm else None
            t0 = time.perf_counter()
            if scene.mode == "pair":
                out = ccd.earliest_contacts(pairs_obj, scene.dt, timings=tm, exhaustive=args.exhaustive)
            else:
                out = ccd._run_problems(problems, widen=1e-3, timings=tm)
            t1 = time.perf_counter()
            if i >= n_warm:
                ms.append(1e3 * (t1 - t0))
        return ms, ph, out

    ccd.set_tree_cache(True)
    e2e_ms, phases, out = e2e_loop(args.warmup, args.steps)
    cold_steps = min(args.steps, 5)
    ccd.set_tree_cache(False)
    cold_ms, cold_phases, _ = e2e_loop(2, cold_steps)
    ccd.set_tree_cache(True)
    clocks.__exit__(None, None, None)
    h2d = float(np.mean(phases.pop("h2d_bytes"))) if phases.get("h2d_bytes") else float(hs.nbytes)
    h2d_cold = float(np.mean(cold_phases.pop("h2d_bytes"))) if cold_phases.get("h2d_bytes") else float(hs.nbytes)
    d2h = sum(v.nbytes for v in out.contacts.values()) + out.dt.nbytes + out.collision.nbytes \
        + out.first_contact.nbytes + out.fused_offset.nbytes

    # ---- reduce over ranks (max time, sum work)
    vals = torch.tensor([total_ms, sum(e2e_ms), float(tests), float(contacts)], dtype=torch.float64,
                        device="cuda")
    if dist is not None:
        t_max = vals[:2].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        w_sum = vals[2:].clone()
        dist.all_reduce(w_sum, op=dist.ReduceOp.SUM)
        total_ms, e2e_total = float(t_max[0]), float(t_max[1])
        tests_all, contacts_all = float(w_sum[0]), float(w_sum[1])
    else:
        e2e_total = sum(e2e_ms)
        tests_all, contacts_all = float(tests), float(contacts)


    if rank == 0:
        value = tests_all / (total_ms * 1e-3)
        # flops of the rows that actually ran the exact 15-feature distance
        # static batches time the exact kernel alone; moving batches run the
        # culls and the exact distance in one kernel (k_screen)
        kern_ms = exact_ms if exact_ms > 0 else screen_ms
        traffic = committed_traffic(args.config, "k_screen_static" if exact_ms > 0 else "k_screen")
        achieved = exact_rows * FLOPS_PER_TEST / (kern_ms * 1e-3) / 1e12 if kern_ms > 0 else 0.0
        line = {
            "metric": METRIC, "value": value, "unit": "tests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": {"workload": args.config + (" exhaustive" if args.exhaustive else ""),
                       "description": CONFIG_DOC[args.config],
                       "problems_per_gpu": len(problems), "pairs_per_gpu": len(hs.pair_problem),
                       "triangle_records_per_gpu": int(hs.n_tris),
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": f"weak: {world} independent shards"},
            "contacts_per_s": contacts_all / (total_ms * 1e-3),
            "tests_per_step": tests_all / args.steps,
            "raw_contacts_per_step": contacts_all / args.steps,
            "e2e": {"value": tests_all / (e2e_total * 1e-3), "unit": "tests/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": e2e_total / args.steps,
                    "path": "ccd.earliest_contacts(host bodies) -> pack -> H2D of the step's states and "
                            "pair tables (surrogate trees device-resident after the first call) -> "
                            "ltsg_search -> D2H",
                    "phases_ms_per_step": {k: sum(v) / len(v) for k, v in phases.items()}},
            "e2e_cold": {"value": tests_all / args.steps * cold_steps / (sum(cold_ms) * 1e-3)
                         if dist is None else None,
                         "unit": "tests/s", "steps": cold_steps,
                         "h2d_bytes_per_step": int(h2d_cold), "ms_per_step": sum(cold_ms) / cold_steps,
                         "path": "as e2e with the device tree cache off: every step also uploads the "
                                 "compact surrogate trees and rebuilds the records on the device",
                         "phases_ms_per_step": {k: sum(v) / len(v) for k, v in cold_phases.items()}},
            "roofline": {"bound": "fp64", "kernel": "k_screen_static" if exact_ms > 0 else "k_screen",
                         "achieved": achieved,
                         "peak": peak_tflops.value, "unit": "TFLOP/s",
                         "frac": achieved / peak_tflops.value if peak_tflops.value else None,
                         "traffic": traffic.get("dram_bytes_per_step"),
                         "traffic_unit": "DRAM bytes per step (sum over the kernel's launches of one search)",
                         "traffic_source": traffic.get("source"),
                         "peak_source": "in-run DFMA microbenchmark (ltsg_fp64_peak); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "flops_per_test": FLOPS_PER_TEST,
                         "kernel_ms_per_step": kern_ms / args.steps,
                         "screen_ms_per_step": screen_ms / args.steps,
                         "expand_ms_per_step": expand_ms / args.steps,
                         "screen_rows_per_step": screen_rows / args.steps,
                         "screen_rows_exact_per_step": exact_rows / args.steps,
                         "note": "rows settled by the certified culls (sphere, separating axes) are "
                                 "counted as tests in `value` (their decision is identical) but not in "
                                 "`achieved`; screen_ms also covers the seeds and the child expansion "
                                 "with its culls (expand_ms)"},
            "roofline_distance_kernel": allpairs,
            "gpu_launches": launches,
            "breakdown_ms_per_step": {
                "screen": screen_ms / args.steps,
                "refine": sum(s.get("ms_refine", 0.0) for s in stats) / args.steps,
                "contacts_fusion": sum(s.get("ms_contacts", 0.0) for s in stats) / args.steps,
                "generations": stats[-1].get("generations"),
                "candidates": stats[-1].get("candidates")},
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "setup_s": t_build,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIG_DOC), default="c1")
    ap.add_argument("--pairs", type=int, default=None, help="override the workload size")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-workers", type=int, default=0)
    ap.add_argument("--exhaustive", action="store_true",
                    help="screen every fine x fine pair (ccd.py:387-388) instead of the multiscale walk")
    ap.add_argument("--no-allpairs", action="store_true", help="skip the distance-kernel roofline leg")
    args = ap.parse_args(argv)
    rank, world, local_rank = _env_rank()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
