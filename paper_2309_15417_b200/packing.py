"""Host packer: reference-shaped inputs -> the device scene of ltsg_search.

Layout in HBM (DESIGN.md §"Data layout"):

* one float64 record of 16 slots (128 B, four 32-B sectors) per surrogate
  triangle of every body and level: the 9 body-frame corners (corner-major),
  epsilon, arm (largest corner norm, ccd._Motion.arm, ccd.py:108-114), the
  (int32 first child, int32 child count) pair in slot 11, and the
  body-frame bounding sphere (centroid, radius; -1 for slivers) in 12..15
  that the certified cull uses.  Levels of a tree
  are re-ordered top-down so that a parent's children (the Morton groups of
  surrogate.py:99-116) are one contiguous range of the finer level: the
  traversal expands children with coalesced, index-free loads.  `tri_orig`
  maps a record back to its index in the reference tree (contacts report it).
* per body: the raw kinematic snapshot (ccd.py:98-106 reads exactly these);
  rotation matrices, spin axes and |omega| are derived on the device with the
  reference's rounding.
* per pair: body slots, problem index and fusion-group rank.

Packed trees are cached per tree object (trees are immutable after
construction), so repeated calls only re-pack states.
"""

from __future__ import annotations

import threading
import weakref
from itertools import chain
from operator import attrgetter, is_not
from dataclasses import dataclass

import numpy as np

MAX_LEVELS = 8
RECORD = 16
CULL_COND = 1e4  # slivers (Lmax^2 > CULL_COND * |e0 x e2|) are never culled


@dataclass
class PackedTree:
    records: np.ndarray      # (n, 16) float64
    orig: np.ndarray         # (n,) int32
    level_off: np.ndarray    # (L,) int64, record offset of each level within the tree
    level_size: np.ndarray   # (L,) int64
    max_children: int
    # compact upload image (ltsg_tree_upload): the device rebuilds `records`
    verts: np.ndarray = None   # (nv, 3) float64 distinct fine-level corners (bitwise)
    vidx: np.ndarray = None    # (n_fine, 3) int32 tree-local vertex ids, record order
    coarse: np.ndarray = None  # (n - n_fine, 9) float64 coarse corners
    eps: np.ndarray = None     # eps_mode 1: (n,); 0: [fine eps, coarse eps...]
    eps_mode: int = 1
    kids: np.ndarray = None    # (n - n_fine, 2) int32 (first child, count)

    @property
    def upload_nbytes(self) -> int:
        return sum(a.nbytes for a in (self.verts, self.vidx, self.coarse, self.eps, self.kids, self.orig))


_cache_lock = threading.Lock()
_cache: dict = {}


def _tree_key(tree):
    return id(tree)


def pack_tree(tree) -> PackedTree:
    """Pack one SurrogateTree (cached by identity while the tree lives)."""
    key = _tree_key(tree)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0]() is tree:
            return hit[1]
    packed = _pack_tree(tree)
    try:
        ref = weakref.ref(tree, lambda _r, k=key: _cache.pop(k, None))
    except TypeError:
        return packed
    with _cache_lock:
        _cache[key] = (ref, packed)
    return packed


def _pack_tree(tree) -> PackedTree:
    levels = tree.levels
    n_levels = len(levels)
    if n_levels < 1:
        raise ValueError("tree has no levels")
    if n_levels > MAX_LEVELS:
        raise ValueError(f"trees deeper than {MAX_LEVELS} levels are not supported")
    # top-down order: perm[l] lists original indices of level l in packed order
    perm = [None] * n_levels
    top = n_levels - 1
    perm[top] = np.arange(levels[top].size, dtype=np.int64)
    first = [None] * n_levels
    count = [None] * n_levels
    max_children = 1
    for lvl in range(top, 0, -1):
        kids = levels[lvl].children
        if kids is None:
            raise ValueError(f"level {lvl} has no children")
        lists = [np.asarray(kids[i], dtype=np.int64) for i in perm[lvl]]
        cnt = np.array([len(k) for k in lists], dtype=np.int64)
        max_children = max(max_children, int(cnt.max()) if len(cnt) else 1)
        order = np.concatenate(lists) if lists else np.zeros(0, dtype=np.int64)
        seen = np.zeros(levels[lvl - 1].size, dtype=bool)
        seen[order] = True
        if not seen.all():  # unreferenced finer triangles: unreachable, keep them anyway
            order = np.concatenate([order, np.flatnonzero(~seen)])
        perm[lvl - 1] = order
        first[lvl] = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
        count[lvl] = cnt
    sizes = np.array([len(p) for p in perm], dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    recs = np.zeros((int(sizes.sum()), RECORD), dtype=np.float64)
    orig = np.empty(int(sizes.sum()), dtype=np.int32)
    for lvl in range(n_levels):
        p = perm[lvl]
        lv = levels[lvl]
        corners = np.asarray(lv.corners, dtype=np.float64)[p]
        sl = slice(offs[lvl], offs[lvl] + sizes[lvl])
        recs[sl, 0:9] = corners.reshape(-1, 9)
        recs[sl, 9] = np.asarray(lv.epsilon, dtype=np.float64)[p]
        # ccd._Motion.arm: np.linalg.norm(corners, axis=2).max(axis=1)
        recs[sl, 10] = np.linalg.norm(corners, axis=2).max(axis=1)
        # body-frame bounding sphere for the certified cull: centroid and
        # radius (slightly inflated), or -1 for slivers
        cen = corners.mean(axis=1)
        rad = np.linalg.norm(corners - cen[:, None, :], axis=2).max(axis=1) * (1.0 + 1e-12)
        e0 = corners[:, 1] - corners[:, 0]
        e2 = corners[:, 2] - corners[:, 0]
        area2 = np.linalg.norm(np.cross(e0, e2), axis=1)
        lmax2 = np.max([np.sum((corners[:, (k + 1) % 3] - corners[:, k]) ** 2, axis=1) for k in range(3)],
                       axis=0)
        ok = (area2 > 0.0) & (lmax2 <= CULL_COND * area2)
        recs[sl, 12:15] = cen
        recs[sl, 15] = np.where(ok, rad, -1.0)
        if lvl > 0:
            ch = np.zeros(len(p), dtype=np.int64)
            ch[: len(first[lvl])] = first[lvl]
            cn = np.zeros(len(p), dtype=np.int64)
            cn[: len(count[lvl])] = count[lvl]
            pair = (ch.astype(np.uint32).astype(np.uint64)
                    | (cn.astype(np.uint32).astype(np.uint64) << np.uint64(32)))
            recs[sl, 11] = pair.view(np.float64)
        orig[sl] = p.astype(np.int32)
    return _with_upload(PackedTree(records=recs, orig=orig, level_off=offs, level_size=sizes,
                                   max_children=max_children))


def _with_upload(pt: PackedTree) -> PackedTree:
    """Attach the compact upload image.  The fine level's corners are rows of
    the mesh vertex array (body.py:70-72), so they are deduplicated on their
    bit patterns (exact, -0.0 kept apart from 0.0)."""
    n0 = int(pt.level_size[0])
    fine = np.ascontiguousarray(pt.records[:n0, :9]).reshape(-1, 3)
    bits = fine.view(np.uint64)
    uniq, inv = np.unique(bits, axis=0, return_inverse=True)
    pt.verts = np.ascontiguousarray(uniq).view(np.float64).reshape(-1, 3)
    pt.vidx = inv.reshape(n0, 3).astype(np.int32)
    pt.coarse = np.ascontiguousarray(pt.records[n0:, :9])
    e = pt.records[:, 9]
    e0 = e[:n0].view(np.uint64)
    if n0 > 0 and np.all(e0 == e0[0]):
        pt.eps_mode = 0
        pt.eps = np.concatenate([e[:1], e[n0:]])
    else:
        pt.eps_mode = 1
        pt.eps = e.copy()
    pt.kids = np.ascontiguousarray(pt.records[n0:, 11]).view(np.int32).reshape(-1, 2).copy()
    return pt


def body_id(body) -> int:
    return int(body.pid) if hasattr(body, "timeline") else int(body.sid)


UPLOAD_KEYS = ("up_verts", "up_vidx", "up_coarse", "up_eps", "up_kids", "up_table")


@dataclass
class HostScene:
    """Packed scene in host (optionally pinned) memory.  The triangle records
    travel as the compact upload image (`up_*`, ltsg_tree_upload) and are
    rebuilt on the device; `records()` assembles them on the host."""
    n_tris: int
    tri_orig: np.ndarray
    body_state: np.ndarray
    body_levels: np.ndarray
    pair_body: np.ndarray
    pair_problem: np.ndarray
    pair_group: np.ndarray
    problem_dt: np.ndarray
    problem_tbase: np.ndarray
    max_children: int
    n_problems: int
    body_ids: np.ndarray
    up_verts: np.ndarray
    up_vidx: np.ndarray
    up_coarse: np.ndarray
    up_eps: np.ndarray
    up_kids: np.ndarray
    up_table: np.ndarray
    trees: list  # the distinct PackedTrees, in table order

    def arrays(self):
        return {k: getattr(self, k) for k in (
            "tri_orig", "body_state", "body_levels", "pair_body", "pair_problem",
            "pair_group", "problem_dt", "problem_tbase") + UPLOAD_KEYS}

    @property
    def nbytes(self) -> int:
        return sum(a.nbytes for a in self.arrays().values())

    def records(self) -> np.ndarray:
        """The (n_tris, 16) records the device rebuilds (host copy, for tests)."""
        return np.concatenate([pt.records for pt in self.trees]) if self.trees else np.zeros((0, RECORD))


def body_state_row(body) -> np.ndarray:
    row = np.zeros(16)
    if hasattr(body, "timeline"):
        s = body.timeline.current
        row[0:3] = np.asarray(s.position, dtype=np.float64)
        row[3:6] = np.asarray(s.velocity, dtype=np.float64)
        row[6:10] = np.asarray(s.rotation, dtype=np.float64)
        row[10:13] = np.asarray(s.angular_velocity, dtype=np.float64)
    else:
        row[13] = 1.0
    return row


class Packer:
    """Re-uses the assembled, pinned tree block across calls that pack the
    same bodies (an engine sweeping the same particles): only the kinematic
    states and the pair tables are rebuilt.  Trees are immutable after
    construction, so the cache is keyed on tree identity."""

    def __init__(self, pinned: bool = True):
        self.pinned = pinned
        self._key = None
        self._static = None

    def pack(self, problems) -> HostScene:
        # problem structure (which body objects pair up how) is cached too:
        # an engine re-screens the same clusters every sweep with new states
        skey = tuple((tuple((id(a), id(b)) for a, b in pairs)) for pairs, _dt, _tb in problems)
        if skey != getattr(self, "_skey", None):
            self._tables = _tables(problems)
            self._skey = skey
        bodies, pair_body, pair_problem, pair_group, _d, _t = self._tables
        dts = np.fromiter((float(dt) for _p, dt, _tb in problems), dtype=np.float64, count=len(problems))
        tbs = np.fromiter((float(tb) for _p, _dt, tb in problems), dtype=np.float64, count=len(problems))
        key = tuple(map(id, map(_TREE, bodies)))
        if key != self._key:
            self._static = _assemble_static(bodies, self.pinned)
            self._key = key
            self._trees = [b.tree for b in bodies]  # keep ids alive while cached
        if getattr(self, "_pair_key", None) is not skey:
            self._pair_arrays = (np.asarray(pair_body, dtype=np.int32).reshape(-1, 2),
                                 np.asarray(pair_problem, dtype=np.int32),
                                 np.asarray(pair_group, dtype=np.int32))
            self._pair_key = skey
        state = self._states(bodies)
        pb, pp, pg = self._pair_arrays
        return _scene(self._static, state, self._ids(bodies, skey), pb, pp, pg, dts, tbs)

    def _ids(self, bodies, skey):
        # body ids and kinds are fixed per body object: cached with the
        # structure (keyed on the body list object, rebuilt with it)
        if getattr(self, "_ids_for", None) is not bodies:
            self._ids_cache = np.fromiter((body_id(b) for b in bodies), dtype=np.int64, count=len(bodies))
            self._dyn_cache = np.flatnonzero(np.fromiter((hasattr(b, "timeline") for b in bodies), dtype=bool,
                                                         count=len(bodies)))
            self._ids_for = bodies
        return self._ids_cache

    def _states(self, bodies):
        # one pinned state buffer, re-used: every search call completes (its
        # results are read back) before the next pack on this thread, so a
        # HostScene from a Packer is valid until the Packer's next pack call
        buf = getattr(self, "_state_buf", None)
        if buf is None or len(buf) != len(bodies):
            buf = _pinned((len(bodies), 16), np.float64) if self.pinned else np.empty((len(bodies), 16))
            self._state_buf = buf
        self._ids(bodies, None)
        return _states(bodies, out=buf, dyn=self._dyn_cache)


    def pack_pairs(self, pairs, dts) -> HostScene:
        """Fast path for pair-mode batches (one body pair per problem, as
        `pair_earliest_contact`): no per-problem Python tuples, one fusion
        group per problem, t_base 0."""
        prev = getattr(self, "_flat", None)
        if prev is not None and getattr(self, "_skey", None) == "pairs" and _fastpack is not None:
            same = _fastpack.pairs_are(pairs, prev)
        else:
            flat = list(chain.from_iterable(pairs))
            same = (prev is not None and len(prev) == len(flat) and getattr(self, "_skey", None) == "pairs"
                    and not any(map(is_not, flat, prev)))
        skey = "pairs"
        if not same:
            self._flat = list(chain.from_iterable(pairs))
            slot_of = {}
            bodies = []
            pb = np.empty((len(pairs), 2), dtype=np.int32)
            for k, (a, b) in enumerate(pairs):
                if body_id(a) == body_id(b):
                    a = b  # the reference's motions dict collapses equal ids to body_b (ccd.py:501)
                for side, x in ((0, a), (1, b)):
                    sl = slot_of.get(id(x))
                    if sl is None:
                        sl = slot_of[id(x)] = len(bodies)
                        bodies.append(x)
                    pb[k, side] = sl
            self._tables = (bodies, pb, np.arange(len(pairs), dtype=np.int32),
                            np.zeros(len(pairs), dtype=np.int32), None, None)
            self._skey = skey
            self._key = None  # force the tree block check below
        bodies, pb, pp, pg, _d, _t = self._tables
        if not (self._key is not None and _fastpack is not None and _fastpack.trees_are(bodies, self._trees)):
            key = tuple(map(id, map(_TREE, bodies)))
            if key != self._key:
                self._static = _assemble_static(bodies, self.pinned)
                self._key = key
                self._trees = [b.tree for b in bodies]
        self._pair_arrays = (pb, pp, pg)
        state = self._states(bodies)
        dts = np.array(np.broadcast_to(np.asarray(dts, dtype=np.float64), (len(pairs),)), copy=True)
        return _scene(self._static, state, self._ids(bodies, skey), pb, pp, pg, dts, np.zeros(len(pairs)))


_TREE = attrgetter("tree")
_CURRENT = attrgetter("timeline.current")
_POS, _VEL, _ROT, _OMEGA = (attrgetter(k) for k in ("position", "velocity", "rotation", "angular_velocity"))


try:  # the C gather of the states (csrc/fastpack.c), built in-tree by build.build_fastpack
    from . import _fastpack
except ImportError:  # pragma: no cover - host packing falls back to numpy
    _fastpack = None


def _states(bodies, out, dyn=None):
    """Body snapshot rows (body_state_row for every body), vectorised.
    `dyn`: indices of the dynamic bodies (computed when not given)."""
    n = len(bodies)
    if _fastpack is not None and out.dtype == np.float64 and out.flags.c_contiguous and out.shape == (n, 16):
        _fastpack.gather_states(bodies, out)
        return out
    state = out
    state.fill(0.0)
    if dyn is None:
        dyn = np.flatnonzero(np.fromiter((hasattr(b, "timeline") for b in bodies), dtype=bool, count=n))
    if len(dyn):
        sel = slice(None) if len(dyn) == n else dyn
        cur = list(map(_CURRENT, bodies if len(dyn) == n else [bodies[i] for i in dyn]))
        # one concatenation per field (C-level iteration over the states)
        for lo, hi, get in ((0, 3, _POS), (3, 6, _VEL), (6, 10, _ROT), (10, 13, _OMEGA)):
            state[sel, lo:hi] = np.concatenate(list(map(get, cur))).reshape(len(cur), hi - lo)
    if len(dyn) < n:
        stat = np.ones(n, dtype=bool)
        stat[dyn] = False
        state[stat, 13] = 1.0
    return state


def _pinned(shape, dtype):
    import torch

    t = torch.empty(shape, dtype={np.float64: torch.float64, np.int32: torch.int32,
                                  np.int64: torch.int64}[dtype], pin_memory=True)
    return t.numpy()


def _tables(problems):
    slot_of = {}
    bodies = []
    pair_body = []
    pair_problem = []
    pair_group = []
    dts = np.empty(len(problems))
    tbs = np.empty(len(problems))
    for pi, (pairs, dt, tb) in enumerate(problems):
        dts[pi] = float(dt)
        tbs[pi] = float(tb)
        ids = []
        for ba, bb in pairs:
            for b in (ba, bb):
                if id(b) not in slot_of:
                    slot_of[id(b)] = len(bodies)
                    bodies.append(b)
            pair_body.append((slot_of[id(ba)], slot_of[id(bb)]))
            pair_problem.append(pi)
            ids.append((body_id(ba), body_id(bb)))
        # fusion groups: distinct (body_a id, body_b id) in sorted order (ccd.py:539)
        uniq = sorted(set(ids))
        rank = {u: r for r, u in enumerate(uniq)}
        pair_group.extend(rank[i] for i in ids)
    return bodies, pair_body, pair_problem, pair_group, dts, tbs


@dataclass
class StaticBlock:
    """The tree part of a scene: compact upload pools, tri_orig, level table."""
    n_tris: int
    orig: np.ndarray
    lev: np.ndarray
    max_children: int
    pools: dict
    trees: list


def _assemble_static(bodies, pinned) -> StaticBlock:
    """Upload image of the bodies' distinct trees + level table."""
    trees = {}
    order = []
    for b in bodies:
        k = id(b.tree)
        if k not in trees:
            trees[k] = pack_tree(b.tree)
            order.append(k)
    pts = [trees[k] for k in order]
    tree_off = {}
    off = 0
    for k in order:
        tree_off[k] = off
        off += len(trees[k].records)
    sizes = {"up_verts": (sum(len(p.verts) for p in pts), 3), "up_vidx": (sum(len(p.vidx) for p in pts), 3),
             "up_coarse": (sum(len(p.coarse) for p in pts), 9), "up_eps": (sum(len(p.eps) for p in pts),),
             "up_kids": (sum(len(p.kids) for p in pts), 2), "up_table": (len(pts), 8)}
    dtypes = {"up_verts": np.float64, "up_vidx": np.int32, "up_coarse": np.float64, "up_eps": np.float64,
              "up_kids": np.int32, "up_table": np.int64}
    pools = {k: (_pinned(sizes[k], dtypes[k]) if pinned else np.empty(sizes[k], dtype=dtypes[k]))
             for k in UPLOAD_KEYS}
    orig = _pinned((off,), np.int32) if pinned else np.empty(off, dtype=np.int32)
    cur = dict.fromkeys(("v", "i", "c", "e"), 0)
    max_children = 1
    for t, k in enumerate(order):
        pt = trees[k]
        n0 = int(pt.level_size[0])
        nv, nc, ne = len(pt.verts), len(pt.coarse), len(pt.eps)
        pools["up_table"][t] = (tree_off[k], n0, nc, cur["v"], cur["i"], cur["c"], cur["e"], pt.eps_mode)
        pools["up_verts"][cur["v"]:cur["v"] + nv] = pt.verts
        pools["up_vidx"][cur["i"]:cur["i"] + n0] = pt.vidx
        pools["up_coarse"][cur["c"]:cur["c"] + nc] = pt.coarse
        pools["up_kids"][cur["c"]:cur["c"] + nc] = pt.kids
        pools["up_eps"][cur["e"]:cur["e"] + ne] = pt.eps
        cur["v"] += nv
        cur["i"] += n0
        cur["c"] += nc
        cur["e"] += ne
        orig[tree_off[k]:tree_off[k] + len(pt.records)] = pt.orig
        max_children = max(max_children, pt.max_children)
    lev = np.zeros((len(bodies), 18), dtype=np.int64)
    for i, b in enumerate(bodies):
        pt = trees[id(b.tree)]
        L = len(pt.level_size)
        lev[i, 0] = L
        lev[i, 2:2 + L] = tree_off[id(b.tree)] + pt.level_off
        lev[i, 10:10 + L] = pt.level_size
    return StaticBlock(n_tris=off, orig=orig, lev=lev, max_children=max_children, pools=pools, trees=pts)


def _scene(static: StaticBlock, state, ids, pair_body, pair_problem, pair_group, dts, tbs) -> HostScene:
    lev = static.lev.copy()
    lev[:, 1] = ids
    return HostScene(
        n_tris=static.n_tris, tri_orig=static.orig, body_state=state, body_levels=lev,
        pair_body=pair_body, pair_problem=pair_problem, pair_group=pair_group,
        problem_dt=dts, problem_tbase=tbs, max_children=static.max_children, n_problems=len(dts),
        body_ids=ids, trees=static.trees, **static.pools)


def pack(problems) -> HostScene:
    """Pack a batch of problems.

    `problems` is a list of (pairs, dt, t_base) where each pair is a tuple of
    two body objects.  A body object shared by several pairs or problems is
    packed once.
    """
    slot_of = {}
    bodies = []
    pair_body = []
    pair_problem = []
    pair_group = []
    dts = np.empty(len(problems))
    tbs = np.empty(len(problems))
    for pi, (pairs, dt, tb) in enumerate(problems):
        dts[pi] = float(dt)
        tbs[pi] = float(tb)
        ids = []
        for ba, bb in pairs:
            for b in (ba, bb):
                if id(b) not in slot_of:
                    slot_of[id(b)] = len(bodies)
                    bodies.append(b)
            pair_body.append((slot_of[id(ba)], slot_of[id(bb)]))
            pair_problem.append(pi)
            ids.append((body_id(ba), body_id(bb)))
        # fusion groups: distinct (body_a id, body_b id) in sorted order (ccd.py:539)
        uniq = sorted(set(ids))
        rank = {u: r for r, u in enumerate(uniq)}
        pair_group.extend(rank[i] for i in ids)
    return _assemble(bodies, pair_body, pair_problem, pair_group, dts, tbs)


def _assemble(bodies, pair_body, pair_problem, pair_group, dts, tbs) -> HostScene:
    static = _assemble_static(bodies, pinned=False)
    state = np.empty((len(bodies), 16))
    for i, b in enumerate(bodies):
        state[i] = body_state_row(b)
    ids = np.fromiter((body_id(b) for b in bodies), dtype=np.int64, count=len(bodies))
    return _scene(static, state, ids,
                  np.asarray(pair_body, dtype=np.int32).reshape(-1, 2),
                  np.asarray(pair_problem, dtype=np.int32), np.asarray(pair_group, dtype=np.int32),
                  np.asarray(dts, dtype=np.float64), np.asarray(tbs, dtype=np.float64))
