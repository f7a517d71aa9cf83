"""Surrogate-tree construction on the GPU.

Drop-in for `ltsdem.surrogate.build_surrogate_tree(mesh, epsilon, fanout=4,
max_levels=8)` (surrogate.py:71-119): same arguments, same errors, same
`SurrogateTree` of `SurrogateLevel`s (children as sorted index arrays), and
the same numbers -- bit for bit with numpy's bundled OpenBLAS/LAPACK, see
csrc/lapack3.cuh.  `build_surrogate_trees` builds many meshes in one call
(every coarse level of every mesh is one Morton-code pass, one radix sort
and one thread per parent group), which is how scene setup uses it.

The computation is the CUDA library's `ltsg_build_trees`; there is no CPU
path (the library raises without a device).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .bodies import ChildIndex, SurrogateLevel, SurrogateTree


def _corners_of(mesh) -> np.ndarray:
    if hasattr(mesh, "corners"):
        corners = np.stack(mesh.corners(), axis=1)
    else:
        corners = np.asarray(mesh, dtype=float).reshape(-1, 3, 3)
    return np.ascontiguousarray(corners, dtype=np.float64)


def level_sizes(n: int, fanout: int = 4, max_levels: int = 8) -> list:
    """Record counts per level (surrogate.py:93-96: coarsen until one root or
    the level cap; each level groups `fanout` records in Morton order)."""
    sizes = [int(n)]
    while sizes[-1] > 1 and len(sizes) < max_levels:
        sizes.append(-(-sizes[-1] // fanout))
    return sizes


class TreeLayout:
    """Where every mesh's levels live in the record table, and the per-level
    step rows the library walks (include/ltsgpu.h, ltsg_tree_build)."""

    def __init__(self, sizes, fanout: int, max_levels: int):
        self.fanout = fanout
        self.levels = [level_sizes(n, fanout, max_levels) for n in sizes]
        counts = np.array([sum(lv) for lv in self.levels], dtype=np.int64)
        self.rec_off = np.zeros(len(sizes) + 1, dtype=np.int64)
        np.cumsum(counts, out=self.rec_off[1:])
        self.n_records = int(self.rec_off[-1])
        self.level_off = []  # per mesh: record offset of each level
        for p, lv in enumerate(self.levels):
            off = np.zeros(len(lv), dtype=np.int64)
            np.cumsum(lv[:-1], out=off[1:])
            self.level_off.append(off + self.rec_off[p])
        depth = max((len(lv) for lv in self.levels), default=1)
        rows, level_steps, level_keys, level_groups = [], [0], [], []
        for lvl in range(1, depth):
            kk = gg = 0
            for p, lv in enumerate(self.levels):
                if len(lv) > lvl:
                    off = self.level_off[p]
                    rows.append((off[lvl - 1], lv[lvl - 1], off[lvl], lv[lvl], kk, gg))
                    kk += lv[lvl - 1]
                    gg += lv[lvl]
            level_steps.append(len(rows))
            level_keys.append(kk)
            level_groups.append(gg)
        self.steps = np.array(rows, dtype=np.int64).reshape(-1, 6)
        self.level_steps = np.array(level_steps, dtype=np.int64)
        self.level_keys = np.array(level_keys, dtype=np.int64)
        self.level_groups = np.array(level_groups, dtype=np.int64)
        self.n_levels = depth - 1


class DeviceTreeBuild:
    """The inputs of one `ltsg_build_trees` call resident on the device:
    `run()` launches the build (idempotent: the fine level is input, the
    coarse levels are rewritten), `fetch()` reads the records back."""

    def __init__(self, corners, eps, fanout: int, max_levels: int, stream=None):
        torch = _lib.require_cuda()
        self.torch = torch
        self.corners = corners
        self.eps = eps
        self.lay = lay = TreeLayout([len(c) for c in corners], fanout, max_levels)
        rec = np.zeros((lay.n_records, 9))
        epsv = np.zeros(lay.n_records)
        for p, c in enumerate(corners):
            o = lay.level_off[p][0]
            rec[o:o + len(c)] = c.reshape(-1, 9)
            epsv[o:o + len(c)] = eps[p]
        self.h2d_bytes = rec.nbytes + epsv.nbytes + lay.steps.nbytes
        dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(self.stream):
            self.d_rec = torch.from_numpy(rec).to(dev, non_blocking=False)
            self.d_eps = torch.from_numpy(epsv).to(dev)
            self.d_kids = torch.full((max(lay.n_records, 1),), -1, dtype=torch.int32, device=dev)
            self.d_steps = torch.from_numpy(lay.steps if len(lay.steps) else np.zeros((1, 6), np.int64)).to(dev)
        self.b = _lib.TreeBuild(rec=self.d_rec.data_ptr(), eps=self.d_eps.data_ptr(), kids=self.d_kids.data_ptr(),
                                steps=self.d_steps.data_ptr(), level_steps=lay.level_steps.ctypes.data,
                                level_keys=lay.level_keys.ctypes.data if lay.n_levels else 0,
                                level_groups=lay.level_groups.ctypes.data if lay.n_levels else 0,
                                n_levels=lay.n_levels, fanout=fanout)
        if lay.n_levels == 0:  # every mesh is a single triangle: nothing to coarsen
            self.b.level_keys = self.b.level_groups = lay.level_steps.ctypes.data

    def run(self) -> None:
        with self.torch.cuda.stream(self.stream):
            _lib.check(_lib.lib().ltsg_build_trees(C.byref(self.b), _lib.workspace().handle,
                                                   C.c_void_p(self.stream.cuda_stream)), "ltsg_build_trees")

    def fetch(self):
        """Read the build back: the coarse records and halos (the fine level
        is the caller's input and is not copied back) and the child index."""
        torch, lay = self.torch, self.lay
        if not hasattr(self, "_coarse_idx"):
            coarse = np.ones(lay.n_records, dtype=bool)
            for p, c in enumerate(self.corners):
                o = lay.level_off[p][0]
                coarse[o:o + len(c)] = False
            self._coarse_pos = np.cumsum(coarse) - 1  # record offset -> row of the coarse read-back
            self._coarse_idx = torch.from_numpy(np.flatnonzero(coarse)).to(self.d_rec.device)
        with torch.cuda.stream(self.stream):
            rec_out = self.d_rec.index_select(0, self._coarse_idx).cpu().numpy()
            eps_out = self.d_eps.index_select(0, self._coarse_idx).cpu().numpy()
            kids_out = self.d_kids.cpu().numpy().astype(np.int64)
        self.d2h_bytes = rec_out.nbytes + eps_out.nbytes + self.d_kids.numel() * 4
        return rec_out, eps_out, kids_out

    def trees(self) -> list:
        rec_out, eps_out, kids_out = self.fetch()
        lay, fanout, pos = self.lay, self.lay.fanout, self._coarse_pos
        trees = []
        for p, c in enumerate(self.corners):
            lv, off = lay.levels[p], lay.level_off[p]
            levels = [SurrogateLevel(corners=c, epsilon=np.full(len(c), float(self.eps[p])), children=None)]
            for l in range(1, len(lv)):
                o, n = int(pos[off[l]]), lv[l]
                fo, fn = off[l - 1], lv[l - 1]
                ptr = np.minimum(np.arange(n + 1, dtype=np.int64) * fanout, fn)
                levels.append(SurrogateLevel(corners=rec_out[o:o + n].reshape(n, 3, 3),
                                             epsilon=eps_out[o:o + n],
                                             children=ChildIndex(ptr, kids_out[fo:fo + fn])))
            trees.append(SurrogateTree(levels=levels))
        return trees


def build_surrogate_trees(meshes, epsilons, fanout: int = 4, max_levels: int = 8,
                          stream=None) -> list:
    """build_surrogate_tree for every (mesh, epsilon) in one device call."""
    _lib.require_cuda()
    corners = [_corners_of(m) for m in meshes]
    eps = np.broadcast_to(np.asarray(epsilons, dtype=np.float64), (len(corners),))
    for e in eps:
        if not e > 0.0:
            raise ValueError(f"epsilon must be positive, got {float(e)}")
    if fanout < 2:
        raise ValueError(f"fanout must be at least 2, got {fanout}")
    if fanout > 8:
        raise ValueError(f"fanout above 8 is not supported by the device builder, got {fanout}")
    if max_levels < 1:
        raise ValueError(f"max_levels must be at least 1, got {max_levels}")
    for c in corners:
        if len(c) == 0:
            raise ValueError("mesh has no triangles")
    job = DeviceTreeBuild(corners, eps, fanout, max_levels, stream)
    job.run()
    return job.trees()


def build_surrogate_tree(mesh, epsilon: float, fanout: int = 4, max_levels: int = 8) -> SurrogateTree:
    """ltsdem.surrogate.build_surrogate_tree (surrogate.py:71-119) on the GPU."""
    if epsilon <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    if fanout < 2:
        raise ValueError(f"fanout must be at least 2, got {fanout}")
    return build_surrogate_trees([mesh], [epsilon], fanout=fanout, max_levels=max_levels)[0]
