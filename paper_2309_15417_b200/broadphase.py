"""Drop-in for `ltsdem.broadphase` backed by the B200 broad-phase kernels.

Same names, arguments, result type and semantics as the reference module
(/root/reference/pkg/src/ltsdem/broadphase.py):

* `TimeStepPolicy(dt_max, growth)`                  broadphase.py:26-43
* `particle_dt(timeline, policy)`                   :46-50
* `pair_window(t1, dt1, t2, dt2)`                   :53-56
* `CollisionGraph(edges, static_links, dts)` with `neighbors()`   :59-70
* `build_collision_graph(particles, statics, policy, exhaustive)` :198-252

`build_collision_graph` packs the bodies' timelines into one record per
particle and runs `ltsg_broadphase` (csrc/broad.cu): trajectories, Check 1
by a sort-and-sweep over the time-collapsed boxes, Check 2 per surviving
pair, all on the device.  The graph is bit-identical to the reference's
(same edges in the same dict order, same windows, links and step bounds).
`exhaustive` is accepted for signature parity; the reference documents that
it changes nothing (:206-207), and the device enumeration is complete either
way.  There is no CPU path: a missing library or device raises.

`particle_dt` and `pair_window` are host scalar helpers the reference's
clustering calls (clustering.py:78); they are restated, not accelerated.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

RECORD = 28  # particle record width (include/ltsgpu.h, ltsg_broad_input)


@dataclass
class TimeStepPolicy:
    """Optimistic per-particle step sizing (broadphase.py:26-43)."""

    dt_max: float
    growth: float = 2.0

    def __post_init__(self) -> None:
        if self.dt_max <= 0.0:
            raise ValueError(f"dt_max must be positive, got {self.dt_max}")
        if self.growth <= 1.0:
            raise ValueError(f"growth must exceed 1, got {self.growth}")


def particle_dt(timeline, policy: TimeStepPolicy) -> float:
    """broadphase.py:46-50."""
    last = timeline.current.t - timeline.old.t
    if last == 0.0:
        return policy.dt_max
    return min(policy.growth * last, policy.dt_max)


def pair_window(t1: float, dt1: float, t2: float, dt2: float) -> tuple:
    """Joint statement window of two particles (broadphase.py:53-56)."""
    start = min(t1, t2)
    return start, start + min(dt1, dt2)


@dataclass
class CollisionGraph:
    edges: dict = field(default_factory=dict)
    static_links: dict = field(default_factory=dict)
    dts: dict = field(default_factory=dict)
    stats: dict = field(default_factory=dict, compare=False)

    def neighbors(self) -> dict:
        adj: dict = {}
        for a, b in self.edges:
            adj.setdefault(a, []).append(b)
            adj.setdefault(b, []).append(a)
        return adj


def _sphere(body):
    """(centre, radius) of a body's bounding sphere: the reference's
    `body.sphere` (body.py:28, :50), or this package's `radius` about the
    mass centre (bodies.Particle)."""
    sph = getattr(body, "sphere", None)
    if sph is not None:
        return np.asarray(sph.center, dtype=np.float64), float(sph.radius)
    return np.zeros(3), float(body.radius)


try:  # the C gather of the records (csrc/fastpack.c), built in-tree by build.build_fastpack
    from . import _fastpack
except ImportError:  # pragma: no cover
    _fastpack = None


def pack_particles(particles: dict, pids=None, out=None) -> np.ndarray:
    """(n, 28) records of the particles in ascending id order."""
    pids = sorted(particles) if pids is None else pids
    if _fastpack is not None:
        rec = np.empty((len(pids), RECORD), dtype=np.float64) if out is None else out
        _fastpack.gather_broad([particles[p] for p in pids], rec)
        return rec
    rec = np.zeros((len(pids), RECORD), dtype=np.float64)
    for k, pid in enumerate(pids):
        p = particles[pid]
        tl = p.timeline
        o, c = tl.old, tl.current
        r = rec[k]
        r[0:3] = o.position
        r[3:7] = o.rotation
        r[7] = o.t
        r[8:11] = c.position
        r[11:15] = c.rotation
        r[15] = c.t
        r[16:19] = c.velocity
        r[19:22] = c.angular_velocity
        centre, radius = _sphere(p)
        r[22:25] = centre
        r[25] = radius
    return rec


def pack_statics(statics: dict, sids=None) -> np.ndarray:
    sids = sorted(statics) if sids is None else sids
    srec = np.zeros((len(sids), 4), dtype=np.float64)
    for k, sid in enumerate(sids):
        centre, radius = _sphere(statics[sid])
        srec[k, 0:3] = centre
        srec[k, 3] = radius
    return srec


@dataclass
class GraphArrays:
    """The graph as arrays (body indices into pids + sids)."""

    dts: np.ndarray
    edge: np.ndarray     # (n_edges, 2) int32 particle indices
    window: np.ndarray   # (n_edges, 2)
    link: np.ndarray     # (n_links, 2) int32 (particle index, static index)
    candidates: int
    ms: float
    launches: int


_cap = [1 << 12]


def graph_arrays(rec: np.ndarray, srec: np.ndarray, policy: TimeStepPolicy, *, workspace=None,
                 device_inputs=None) -> GraphArrays:
    """ltsg_broadphase on packed records.  `device_inputs` may hold the two
    record arrays already on the device (torch tensors)."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    n_p, n_s = len(rec), len(srec)
    if device_inputs is not None:
        d_rec, d_srec = device_inputs
    else:
        d_rec = torch.from_numpy(np.ascontiguousarray(rec, dtype=np.float64)).to(dev, non_blocking=True)
        d_srec = torch.from_numpy(np.ascontiguousarray(srec, dtype=np.float64)).to(dev, non_blocking=True)
    ws = workspace or _lib.workspace()
    st = torch.cuda.current_stream()
    dts = torch.empty(max(n_p, 1), dtype=torch.float64, device=dev)
    inp = _lib.BroadInput(particle=d_rec.data_ptr() if n_p else 0, statics=d_srec.data_ptr() if n_s else 0,
                          n_particles=n_p, n_statics=n_s, dt_max=float(policy.dt_max),
                          growth=float(policy.growth))
    cap = _cap[0]
    while True:
        edge = torch.empty((cap, 2), dtype=torch.int32, device=dev)
        window = torch.empty((cap, 2), dtype=torch.float64, device=dev)
        link = torch.empty((cap, 2), dtype=torch.int32, device=dev)
        out = _lib.BroadOutput(dts=dts.data_ptr(), edge=edge.data_ptr(), window=window.data_ptr(),
                               link=link.data_ptr(), cap_edges=cap, cap_links=cap)
        rc = _lib.lib().ltsg_broadphase(C.byref(inp), C.byref(out), ws.handle, C.c_void_p(st.cuda_stream))
        if rc == _lib.LTSG_ECAPACITY and max(out.n_edges, out.n_links) > cap:
            cap = int(max(out.n_edges, out.n_links) * 1.25) + 16
            _cap[0] = max(_cap[0], cap)
            continue
        _lib.check(rc, "ltsg_broadphase")
        break
    ne, nl = int(out.n_edges), int(out.n_links)
    return GraphArrays(dts=dts[:n_p].cpu().numpy(), edge=edge[:ne].cpu().numpy(), window=window[:ne].cpu().numpy(),
                       link=link[:nl].cpu().numpy(), candidates=int(out.candidates), ms=float(out.ms),
                       launches=int(out.launches))


def build_collision_graph(particles: dict, statics: dict, policy: TimeStepPolicy,
                          exhaustive: bool = False) -> CollisionGraph:
    """Run both checks over all candidate pairs and record survivors
    (broadphase.py:198-252), on the GPU."""
    pids = sorted(particles)
    sids = sorted(statics)
    if not pids:
        return CollisionGraph()
    ga = graph_arrays(pack_particles(particles, pids), pack_statics(statics, sids), policy)
    graph = CollisionGraph(dts=dict(zip(pids, ga.dts.tolist())))
    pid_arr = np.asarray(pids)
    ea, eb = pid_arr[ga.edge[:, 0]].tolist(), pid_arr[ga.edge[:, 1]].tolist()
    graph.edges = dict(zip(zip(ea, eb), map(tuple, ga.window.tolist())))
    links: dict = {}
    sid_arr = np.asarray(sids)
    for p, s in zip(pid_arr[ga.link[:, 0]].tolist(), sid_arr[ga.link[:, 1]].tolist()):
        links.setdefault(p, []).append(s)
    graph.static_links = {p: tuple(v) for p, v in links.items()}
    graph.stats = {"candidates": ga.candidates, "ms": ga.ms, "launches": ga.launches}
    return graph


def tube_rows(t1, c1, r1, t2, c2, r2, window, nt1=None, nt2=None):
    """check_spacetime_tube (:154-158) on explicit trajectory rows; returns
    (minimum centre distance, verdict) per row."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    n = len(window)
    if n == 0:
        return np.zeros(0), np.zeros(0, dtype=bool)

    def d(x, dtype=np.float64):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=dtype)).to(dev)

    nt1 = np.full(n, 3) if nt1 is None else nt1
    nt2 = np.full(n, 3) if nt2 is None else nt2
    args = [d(t1), d(c1), d(r1), d(nt1, np.int32), d(t2), d(c2), d(r2), d(nt2, np.int32), d(window)]
    dist = torch.empty(n, dtype=torch.float64, device=dev)
    hit = torch.empty(n, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    rc = _lib.lib().ltsg_tube_rows(*[C.c_void_p(a.data_ptr()) for a in args], n, C.c_void_p(dist.data_ptr()),
                                   C.c_void_p(hit.data_ptr()), C.c_void_p(st.cuda_stream))
    _lib.check(rc, "ltsg_tube_rows")
    return dist.cpu().numpy(), hit.cpu().numpy() != 0
