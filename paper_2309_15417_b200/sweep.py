"""Batched per-sweep narrow phase.

The reference engine sizes every cluster of a sweep with one
`compute_effective_dt` call per uncached cluster, fanned out over a thread
pool (`ltsdem/engine.py:168-200`), and reuses the previous outcome of a
cluster whose inputs did not move (`_cache_key`, engine.py:119-121,
:175-182).  `SweepDriver` keeps exactly that cache and replaces the per-
cluster calls by ONE batched device launch over all uncached clusters
(`ccd.effective_dts`: the clusters are independent problems of one
`ltsg_search`, each with its own shared bound, ccd.py:505-524).

Integration into `ltsdem.engine.step` (INTEGRATION.md shows the patch): the
`jobs` loop becomes

    driver.results(clusters, particles, world.statics,
                   pairs_of=lambda i: _cluster_pairs(clusters[i], graph))

and `solve_impulses` then runs per cluster on the returned contacts, as in
`_compute_cluster` (engine.py:137-143).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import ccd


def cache_key(cluster, particles) -> tuple:
    """The engine's cache key (engine.py:119-121): members, window, statics
    and the members' timeline versions."""
    versions = tuple(particles[pid].timeline.version for pid in cluster.members)
    return (tuple(cluster.members), cluster.t_current, cluster.dt, tuple(getattr(cluster, "statics", ())), versions)


@dataclass
class SweepStats:
    clusters: int = 0
    computed: int = 0   # clusters sized by this sweep's launch
    reused: int = 0     # clusters whose cached outcome was reused
    launches: int = 0   # batched device calls (0 or 1)


class SweepDriver:
    """Per-sweep cluster results with the engine's result cache.

    `results()` returns one NarrowResult per cluster (same order).  Clusters
    whose cache key matches an outcome kept from the previous sweep reuse it;
    all others are computed in one batched launch.  As in the engine, only
    the previous sweep's outcomes are kept (engine.py:208-243 rebuilds the
    cache every sweep; a committed cluster's versions change, so its key
    cannot match again)."""

    def __init__(self, widen: float = ccd._WIDEN):
        self.widen = widen
        self._cache: dict[tuple, ccd.NarrowResult] = {}
        self.last = SweepStats()

    def results(self, clusters, particles, statics, pairs_of, keep=None) -> list:
        """`pairs_of(i)` gives cluster i's body-id pairs (only called for the
        clusters that are computed, like engine._cluster_pairs).  `keep(i)`
        (default: keep all) selects whose outcomes stay cached for the next
        sweep."""
        clusters = list(clusters)
        keys = [cache_key(c, particles) for c in clusters]
        out = [self._cache.get(k) for k in keys]
        todo = [i for i, r in enumerate(out) if r is None]
        stats = SweepStats(clusters=len(clusters), computed=len(todo), reused=len(clusters) - len(todo))
        if todo:
            got, batch = ccd.effective_dts([clusters[i] for i in todo], particles, statics,
                                           [list(pairs_of(i)) for i in todo], widen=self.widen)
            stats.launches = 1 if batch is not None else 0
            for i, r in zip(todo, got):
                out[i] = r
        self._cache = {k: r for i, (k, r) in enumerate(zip(keys, out)) if keep is None or keep(i)}
        self.last = stats
        return out
