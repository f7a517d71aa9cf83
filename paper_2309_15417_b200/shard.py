"""Multi-GPU sharding of the narrow phase: one process per GPU, no data-path
collective.

Narrow-phase problems are independent (each `pair_earliest_contact` call,
each `compute_effective_dt` cluster, engine.py:170-199), so N GPUs split the
problems of a sweep into N contiguous, work-balanced shards and run them
with no communication.  The only exchange is host-side bookkeeping after
the fact (gathering per-problem results for the caller), done with
`torch.distributed.all_gather_object` on whatever backend the job uses
(NCCL on the GPU box, gloo in the CPU tests).  SURVEY.md §8(e).
"""

from __future__ import annotations

import numpy as np


def problem_weights(problems) -> np.ndarray:
    """Work estimate per problem: sum over its pairs of fine-triangle products."""
    w = np.empty(len(problems))
    for i, (pairs, _dt, _tb) in enumerate(problems):
        w[i] = sum(float(a.tree.levels[0].size) * float(b.tree.levels[0].size) for a, b in pairs)
    return w


def shard_bounds(weights, rank: int, world: int):
    """Contiguous [lo, hi) of the problems owned by `rank`, balancing the
    cumulative weight; every problem is owned by exactly one rank."""
    weights = np.asarray(weights, dtype=np.float64)
    n = len(weights)
    if world <= 1 or n == 0:
        return 0, n
    cum = np.concatenate([[0.0], np.cumsum(weights)])
    total = cum[-1]
    if total <= 0.0:
        cuts = [round(n * r / world) for r in range(world + 1)]
    else:
        cuts = [0] + [int(np.searchsorted(cum, total * r / world, side="left")) for r in range(1, world)] + [n]
        cuts = list(np.maximum.accumulate(np.clip(cuts, 0, n)))
    return int(cuts[rank]), int(cuts[rank + 1])


def run_shard(problems, rank: int, world: int, run, weights=None):
    """Run `run(problems[lo:hi])` for this rank's shard; returns (lo, hi, out)."""
    w = problem_weights(problems) if weights is None else weights
    lo, hi = shard_bounds(w, rank, world)
    return lo, hi, run(problems[lo:hi]) if hi > lo else None


def gather_results(local_results, lo: int, n_total: int, group=None):
    """All-gather per-problem results (host objects) and reassemble them in
    problem order on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, list(local_results)), group=group)
    out = [None] * n_total
    for start, res in parts:
        for k, r in enumerate(res):
            out[start + k] = r
    missing = [i for i, r in enumerate(out) if r is None]
    if missing:
        raise RuntimeError(f"problems {missing[:5]} were not computed by any rank")
    return out
