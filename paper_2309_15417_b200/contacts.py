"""Drop-in for `ltsdem.contacts` backed by the B200 contact-consumer kernels.

Same names, arguments, result type and semantics as the reference module
(/root/reference/pkg/src/ltsdem/contacts.py):

* `SolverConfig`, `ImpulseSolution`                       contacts.py:25-55
* `color_contact_graph(contacts)`                          :58-78
* `solve_impulses(contacts, particles, config)`            :114-198
* `integrate_cluster(cluster, particles, result, solution)` :225-253
* `apply_separation(contacts, particles, beta)`            :256-285

plus batched forms a sweep driver uses to put every cluster of a sweep on
the GPU in one launch (`solve_batch`, `integrate_batch`).  Each call runs
the sm_100a kernels of csrc/contacts.cu through the C ABI
(`ltsg_solve_impulses`, `ltsg_integrate`): one warp per cluster, the
sequential-impulse sweeps run class by class with a class's contacts
spread over the lanes.  Results are bit-identical to the reference for
bodies without spin; with spin, `quaternions.advance`'s sin/cos (CUDA vs
libm) can differ in the last bit.  `color_contact_graph` is a host
restatement (the kernels colour on the device themselves).  There is no CPU
path: a missing library or device raises.

Particles are duck-typed like the reference's: `timeline.current`
(position, velocity, rotation, angular_velocity, t), `timeline.new`,
`timeline.touch()`, `mass.mass` and `mass.inverse_inertia` (body frame).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

BODY = 24  # body record width (include/ltsgpu.h, ltsg_solve_input)
STATE = 14  # new-snapshot width (ltsg_integrate)


@dataclass
class SolverConfig:
    restitution: float = 1.0
    friction: float = 0.3
    relaxation: float = 0.5
    penalty: float = 1.0
    threshold: float = 1e-4
    max_iterations: int = 256
    beta: float = 0.2

    def __post_init__(self) -> None:
        if not 0.0 <= self.restitution <= 1.0:
            raise ValueError(f"restitution must be in [0, 1], got {self.restitution}")
        if self.friction < 0.0:
            raise ValueError(f"friction must be >= 0, got {self.friction}")
        if not 0.0 < self.relaxation <= 1.0:
            raise ValueError(f"relaxation must be in (0, 1], got {self.relaxation}")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be positive")


@dataclass
class ImpulseSolution:
    """Post-impulse velocities for every dynamic body that was touched."""

    velocities: dict
    angular_velocities: dict
    iterations: int
    converged: bool
    normal_impulses: list = field(default_factory=list)
    friction_impulses: list = field(default_factory=list)


def color_contact_graph(contacts) -> list:
    """Greedy colour classes: no class reuses a dynamic body (contacts.py:58-78)."""
    classes: list = []
    used: list = []
    for idx, c in enumerate(contacts):
        bodies = {bid for bid in (c.body_a, c.body_b) if bid >= 0}
        for k, taken in enumerate(used):
            if not taken & bodies:
                classes[k].append(idx)
                taken |= bodies
                break
        else:
            classes.append([idx])
            used.append(set(bodies))
    return classes


def body_record(p) -> np.ndarray:
    s = p.timeline.current
    r = np.empty(BODY, dtype=np.float64)
    r[0:3] = s.position
    r[3:6] = s.velocity
    r[6:10] = s.rotation
    r[10:13] = s.angular_velocity
    r[13] = s.t
    r[14] = 1.0 / p.mass.mass
    r[15:24] = np.asarray(p.mass.inverse_inertia, dtype=np.float64).reshape(9)
    return r


def _dev():
    torch = _lib.require_cuda()
    return torch, torch.device("cuda", torch.cuda.current_device())


def _d(torch, dev, x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=dtype)).to(dev, non_blocking=True)


class _Packed:
    """Bodies and contacts of several clusters as the ABI's arrays."""

    def __init__(self, contact_lists, particles, extra_ids=()):
        self.index: dict = {}
        ids = []
        for contacts in contact_lists:
            for c in contacts:
                for bid in (c.body_a, c.body_b):
                    if bid >= 0 and bid not in self.index:
                        self.index[bid] = len(ids)
                        ids.append(bid)
        for bid in extra_ids:
            if bid not in self.index:
                self.index[bid] = len(ids)
                ids.append(bid)
        self.ids = ids
        self.body = np.array([body_record(particles[b]) for b in ids], dtype=np.float64).reshape(-1, BODY)
        n = sum(len(cl) for cl in contact_lists)
        self.offset = np.zeros(len(contact_lists) + 1, dtype=np.int64)
        self.offset[1:] = np.cumsum([len(cl) for cl in contact_lists])
        self.side = np.empty((n, 2), dtype=np.int32)
        self.id = np.empty((n, 2), dtype=np.int64)
        self.position = np.empty((n, 3))
        self.normal = np.empty((n, 3))
        self.t = np.empty(n)
        self.depth = np.empty(n)
        k = 0
        for contacts in contact_lists:
            for c in contacts:
                self.id[k] = (c.body_a, c.body_b)
                self.side[k] = (self.index[c.body_a] if c.body_a >= 0 else -1,
                                self.index[c.body_b] if c.body_b >= 0 else -1)
                self.position[k] = c.position
                self.normal[k] = c.normal
                self.t[k] = c.t
                self.depth[k] = c.depth
                k += 1
        self.n = n

    def check_times(self):
        """extrapolate_free_flight refuses to fly backwards (state.py:91-92)."""
        for k in range(self.n):
            for s in (0, 1):
                b = self.side[k, s]
                if b >= 0 and self.t[k] - self.body[b, 13] < 0.0:
                    raise ValueError(f"free flight requires dt >= 0, got {self.t[k] - self.body[b, 13]}")


def solve_arrays(body, side, position, normal, t, offset, config: SolverConfig, *, workspace=None):
    """ltsg_solve_impulses on packed arrays; returns a dict of host arrays."""
    torch, dev = _dev()
    n_b, n_c, n_p = len(body), len(t), len(offset) - 1
    d = {k: _d(torch, dev, v, dt) for k, v, dt in (
        ("body", body, np.float64), ("side", side, np.int32), ("position", position, np.float64),
        ("normal", normal, np.float64), ("t", t, np.float64), ("offset", offset, np.int64))}
    vel = torch.empty((max(n_b, 1), 3), dtype=torch.float64, device=dev)
    ang = torch.empty((max(n_b, 1), 3), dtype=torch.float64, device=dev)
    touched = torch.zeros(max(n_b, 1), dtype=torch.int32, device=dev)
    lam = torch.empty(max(n_c, 1), dtype=torch.float64, device=dev)
    fric = torch.empty((max(n_c, 1), 3), dtype=torch.float64, device=dev)
    color = torch.empty(max(n_c, 1), dtype=torch.int32, device=dev)
    iters = torch.empty(max(n_p, 1), dtype=torch.int32, device=dev)
    conv = torch.empty(max(n_p, 1), dtype=torch.int32, device=dev)
    inp = _lib.SolveInput(
        body=d["body"].data_ptr() if n_b else 0, n_bodies=n_b, n_problems=n_p,
        contact_offset=d["offset"].data_ptr(), side=d["side"].data_ptr() if n_c else 0,
        position=d["position"].data_ptr() if n_c else 0, normal=d["normal"].data_ptr() if n_c else 0,
        t=d["t"].data_ptr() if n_c else 0, n_contacts=n_c, restitution=float(config.restitution),
        friction=float(config.friction), relaxation=float(config.relaxation), penalty=float(config.penalty),
        threshold=float(config.threshold), max_iterations=int(config.max_iterations))
    out = _lib.SolveOutput(velocity=vel.data_ptr(), angular_velocity=ang.data_ptr(), touched=touched.data_ptr(),
                           normal_impulse=lam.data_ptr(), friction_impulse=fric.data_ptr(), color=color.data_ptr(),
                           iterations=iters.data_ptr(), converged=conv.data_ptr())
    ws = workspace or _lib.workspace()
    st = torch.cuda.current_stream()
    _lib.check(_lib.lib().ltsg_solve_impulses(C.byref(inp), C.byref(out), ws.handle, C.c_void_p(st.cuda_stream)),
               "ltsg_solve_impulses")
    return {"velocity": vel[:n_b].cpu().numpy(), "angular_velocity": ang[:n_b].cpu().numpy(),
            "touched": touched[:n_b].cpu().numpy() != 0, "normal_impulse": lam[:n_c].cpu().numpy(),
            "friction_impulse": fric[:n_c].cpu().numpy(), "color": color[:n_c].cpu().numpy(),
            "iterations": iters[:n_p].cpu().numpy(), "converged": conv[:n_p].cpu().numpy() != 0,
            "ms": float(out.ms), "launches": int(out.launches)}


def solve_batch(contact_lists, particles, config: SolverConfig | None = None) -> list:
    """`solve_impulses` for the clusters of one sweep in one launch.  A dynamic
    body may appear in one cluster's contacts only."""
    cfg = config or SolverConfig()
    contact_lists = [list(cl) for cl in contact_lists]
    if not any(contact_lists):
        return [ImpulseSolution({}, {}, 0, True) for _ in contact_lists]
    pk = _Packed(contact_lists, particles)
    owner: dict = {}
    for p, cl in enumerate(contact_lists):
        for c in cl:
            for bid in (c.body_a, c.body_b):
                if bid >= 0 and owner.setdefault(bid, p) != p:
                    raise ValueError(f"body {bid} appears in the contacts of two clusters")
    pk.check_times()
    r = solve_arrays(pk.body, pk.side, pk.position, pk.normal, pk.t, pk.offset, cfg)
    out = []
    for p, cl in enumerate(contact_lists):
        if not cl:
            out.append(ImpulseSolution({}, {}, 0, True))
            continue
        vel, ang = {}, {}
        for c in cl:  # the reference's dict order: first appearance, side a then b
            for bid in (c.body_a, c.body_b):
                if bid >= 0 and bid not in vel:
                    i = pk.index[bid]
                    vel[bid] = r["velocity"][i].copy()
                    ang[bid] = r["angular_velocity"][i].copy()
        lo, hi = int(pk.offset[p]), int(pk.offset[p + 1])
        out.append(ImpulseSolution(
            velocities=vel, angular_velocities=ang, iterations=int(r["iterations"][p]),
            converged=bool(r["converged"][p]),
            normal_impulses=[float(x) for x in r["normal_impulse"][lo:hi]],
            friction_impulses=[f.copy() for f in r["friction_impulse"][lo:hi]]))
    return out


def solve_impulses(contacts, particles, config: SolverConfig | None = None) -> ImpulseSolution:
    """Resolve all contacts at once, returning post-impulse velocities (contacts.py:114-198)."""
    contacts = list(contacts)
    if not contacts:
        return ImpulseSolution({}, {}, 0, True)
    return solve_batch([contacts], particles, config)[0]


def _new_state(tl, row):
    return type(tl.current)(row[0:3].copy(), row[3:6].copy(), row[6:10].copy(), row[10:13].copy(), float(row[13]))


def integrate_batch(clusters, particles, results, solutions, beta: float | None = None) -> None:
    """`integrate_cluster` then (with `beta`) `apply_separation` of each
    cluster's committed contacts -- the engine's commit of a sweep's active
    clusters (engine.py:283-284) -- in one launch."""
    torch, dev = _dev()
    clusters, results, solutions = list(clusters), list(results), list(solutions)
    contact_lists = [list(r.contacts) for r in results]
    members = [list(c.members) for c in clusters]
    pk = _Packed(contact_lists, particles, extra_ids=[m for ms in members for m in ms])
    n_p = len(clusters)
    moff = np.zeros(n_p + 1, dtype=np.int64)
    moff[1:] = np.cumsum([len(m) for m in members])
    member = np.array([pk.index[m] for ms in members for m in ms], dtype=np.int32)
    t_new = np.array([c.t_current + r.dt for c, r in zip(clusters, results)], dtype=np.float64)
    n_b = len(pk.ids)
    vel = np.zeros((n_b, 3))
    ang = np.zeros((n_b, 3))
    touched = np.zeros(n_b, dtype=np.int32)
    for sol in solutions:
        if sol is None:
            continue
        for bid, v in sol.velocities.items():
            i = pk.index.get(bid)
            if i is not None:
                vel[i] = v
                ang[i] = sol.angular_velocities[bid]
                touched[i] = 1
    for k in range(pk.n):  # extrapolate_free_flight refuses to fly backwards (state.py:91-92)
        for s in (0, 1):
            b = pk.side[k, s]
            if b >= 0 and touched[b] and pk.t[k] - pk.body[b, 13] < 0.0:
                raise ValueError(f"free flight requires dt >= 0, got {pk.t[k] - pk.body[b, 13]}")
    _integrate(torch, dev, pk, moff, member, t_new, vel, ang, touched, 0.0 if beta is None else beta,
               separate=beta is not None, new_in=None, write=lambda b, row: _commit(particles[b], row))


def _commit(p, row):
    tl = p.timeline
    tl.new = _new_state(tl, row)
    tl.touch()


def integrate_arrays(body, member_offset, member, t_new, offset, side, ids, normal, t, depth, vel=None, ang=None,
                     touched=None, beta=0.0, separate=False, new_in=None):
    """ltsg_integrate on packed arrays; returns the (n_bodies, 14) new-snapshot
    rows (rows of non-members are zero)."""
    torch, dev = _dev()
    n_b, n_c = len(body), len(t)
    d = lambda x, dt: _d(torch, dev, x, dt)  # noqa: E731
    dbody, coff = d(body, np.float64), d(offset, np.int64)
    arrs = [d(x, dt) for x, dt in ((side, np.int32), (ids, np.int64), (normal, np.float64), (t, np.float64),
                                     (depth, np.float64))]
    dm, dmo, dtn = d(member, np.int32), d(member_offset, np.int64), d(t_new, np.float64)
    sol = touched is not None and bool(np.any(touched))
    dv = d(vel, np.float64) if sol else None
    da = d(ang, np.float64) if sol else None
    dtch = d(touched, np.int32) if sol else None
    dnew = d(new_in, np.float64) if new_in is not None else None
    out = torch.zeros((max(n_b, 1), STATE), dtype=torch.float64, device=dev)
    inp = _lib.IntegrateInput(
        body=dbody.data_ptr(), n_bodies=n_b, n_problems=len(member_offset) - 1, member_offset=dmo.data_ptr(),
        member=dm.data_ptr(), t_new=dtn.data_ptr(), contact_offset=coff.data_ptr(),
        side=arrs[0].data_ptr() if n_c else 0, id=arrs[1].data_ptr() if n_c else 0,
        normal=arrs[2].data_ptr() if n_c else 0, t=arrs[3].data_ptr() if n_c else 0,
        depth=arrs[4].data_ptr() if n_c else 0, n_contacts=n_c,
        velocity=dv.data_ptr() if sol else 0, angular_velocity=da.data_ptr() if sol else 0,
        touched=dtch.data_ptr() if sol else 0, beta=float(beta),
        new_state_in=dnew.data_ptr() if dnew is not None else 0, separate=1 if separate else 0)
    st = torch.cuda.current_stream()
    _lib.check(_lib.lib().ltsg_integrate(C.byref(inp), C.c_void_p(out.data_ptr()), _lib.workspace().handle,
                                         C.c_void_p(st.cuda_stream)), "ltsg_integrate")
    return out[:n_b].cpu().numpy()


def _integrate(torch, dev, pk, moff, member, t_new, vel, ang, touched, beta, separate, new_in, write):
    host = integrate_arrays(pk.body, moff, member, t_new, pk.offset, pk.side, pk.id, pk.normal, pk.t, pk.depth,
                            vel, ang, touched, beta, separate, new_in)
    for i in member:
        write(pk.ids[i], host[i])
    return host


def integrate_cluster(cluster, particles, result, solution) -> None:
    """Write prospective new snapshots for every cluster member (contacts.py:225-253)."""
    integrate_batch([cluster], particles, [result], [solution], beta=None)


def apply_separation(contacts, particles, beta: float) -> None:
    """Push overlapping pairs apart on their new snapshots (contacts.py:256-285)."""
    torch, dev = _dev()
    contacts = list(contacts)
    pushes = sorted({(c.body_a, c.body_b) for c in contacts if c.depth > 0.0})
    if not pushes:
        return
    pk = _Packed([contacts], particles)
    live = [b for b in pk.ids if particles[b].timeline.new is not None]
    if not live:
        return
    new_in = np.zeros((len(pk.ids), STATE))
    for b in live:
        s = particles[b].timeline.new
        i = pk.index[b]
        new_in[i, 0:3], new_in[i, 3:6], new_in[i, 6:10], new_in[i, 10:13], new_in[i, 13] = \
            s.position, s.velocity, s.rotation, s.angular_velocity, s.t
    member = np.array([pk.index[b] for b in live], dtype=np.int32)
    moff = np.array([0, len(member)], dtype=np.int64)
    # the reference touches a timeline once per body pair that moves it
    touches: dict = {}
    for a, b in pushes:
        wa = 1.0 / particles[a].mass.mass if a >= 0 else 0.0
        wb = 1.0 / particles[b].mass.mass if b >= 0 else 0.0
        if wa + wb == 0.0:
            continue
        for x in (a, b):
            if x >= 0:
                touches[x] = touches.get(x, 0) + 1

    def write(bid, row):
        if bid not in touches:
            return
        tl = particles[bid].timeline
        tl.new.position = row[0:3].copy()
        for _ in range(touches[bid]):
            tl.touch()

    _integrate(torch, dev, pk, moff, member, np.zeros(1), np.zeros((len(pk.ids), 3)), np.zeros((len(pk.ids), 3)),
               np.zeros(len(pk.ids), dtype=np.int32), beta, separate=True, new_in=new_in, write=write)
