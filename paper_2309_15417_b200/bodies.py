"""Input structures of the narrow phase, duck-type compatible with `ltsdem`.

The drop-in API (`ccd.py`) reads exactly the fields the reference's
`ccd._Motion.of_body` reads (ccd.py:98-106):

* dynamic particle: `pid`, `tree`, `timeline.current.{position, velocity,
  rotation, angular_velocity}` (body.py:21-41, state.py:29-46);
* static body: `sid` (negative), `tree` (body.py:44-53);
* tree: `levels[l].{corners (k,3,3), epsilon (k,), children}` with level 0
  the fine mesh (surrogate.py:23-46);
* cluster: `dt`, `t_current` (clustering.py:19-34).

So reference `Particle` / `StaticBody` objects can be passed in unchanged.
The light classes here exist so the GPU box -- where the reference is not
installed -- can build the same inputs.  Constructing them (mass
properties, recentring, tree building) is host setup, not the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class SurrogateLevel:
    corners: np.ndarray                 # (k, 3, 3) body-frame corners
    epsilon: np.ndarray                 # (k,) halo width
    children: list | None               # sorted index arrays into the finer level

    @property
    def size(self) -> int:
        return len(self.corners)


class ChildIndex:
    """Children of one surrogate level as a CSR index.  Behaves like the
    reference's list of sorted index arrays (surrogate.py:115):
    `children[i]` is parent i's child indices, `len`, iteration."""

    __slots__ = ("ptr", "idx")

    def __init__(self, ptr, idx):
        self.ptr = np.asarray(ptr, dtype=np.int64)
        self.idx = np.asarray(idx, dtype=np.int64)

    def __len__(self):
        return len(self.ptr) - 1

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self.idx[self.ptr[i]:self.ptr[i + 1]]

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


@dataclass
class SurrogateTree:
    levels: list                        # levels[0] fine ... levels[-1] coarsest

    @property
    def depth(self) -> int:
        return len(self.levels)

    def level_sizes(self) -> list:
        return [lvl.size for lvl in self.levels]


@dataclass
class ParticleState:
    position: np.ndarray
    velocity: np.ndarray
    rotation: np.ndarray                # unit quaternion [w, x, y, z]
    angular_velocity: np.ndarray        # world frame
    t: float = 0.0


@dataclass
class ParticleTimeline:
    old: ParticleState
    current: ParticleState
    new: ParticleState | None = None
    version: int = field(default=0, compare=False)

    def touch(self) -> None:
        """Bumped on every mutation so caches keyed on timelines stay honest (state.py:70-75)."""
        self.version += 1


@dataclass
class BoundingSphere:
    center: np.ndarray
    radius: float                       # includes the epsilon halo


@dataclass
class Particle:
    pid: int
    tree: SurrogateTree
    epsilon: float
    radius: float                       # bounding-sphere radius about the COM, incl. epsilon
    timeline: ParticleTimeline

    @property
    def sphere(self) -> BoundingSphere:
        """make_particle pins the sphere at the mass centre (body.py:73-83)."""
        return BoundingSphere(center=np.zeros(3), radius=self.radius)


@dataclass
class StaticBody:
    sid: int                            # negative
    tree: SurrogateTree
    epsilon: float
    sphere: BoundingSphere | None = None  # world frame (body.py:50); the broad phase reads it


@dataclass
class Cluster:
    members: tuple
    t_current: float = 0.0
    dt: float = 0.0
    statics: tuple = ()


def state(position, velocity=(0.0, 0.0, 0.0), rotation=(1.0, 0.0, 0.0, 0.0),
          angular_velocity=(0.0, 0.0, 0.0), t=0.0) -> ParticleState:
    return ParticleState(
        position=np.asarray(position, dtype=np.float64).copy(),
        velocity=np.asarray(velocity, dtype=np.float64).copy(),
        rotation=np.asarray(rotation, dtype=np.float64).copy(),
        angular_velocity=np.asarray(angular_velocity, dtype=np.float64).copy(),
        t=float(t),
    )


def timeline(st: ParticleState) -> ParticleTimeline:
    return ParticleTimeline(old=_copy(st), current=_copy(st))


def _copy(st: ParticleState) -> ParticleState:
    return ParticleState(st.position.copy(), st.velocity.copy(), st.rotation.copy(),
                         st.angular_velocity.copy(), st.t)


def centre_of_mass(vertices: np.ndarray, triangles: np.ndarray) -> np.ndarray:
    """Signed-tetrahedron centre of mass of a closed mesh (mesh.py:300-316)."""
    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles, dtype=np.int64)
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    dets = np.einsum("ij,ij->i", a, np.cross(b, c))
    volume = dets.sum() / 6.0
    if volume <= 0.0:
        raise ValueError(f"mesh encloses non-positive volume {volume}")
    return (dets[:, None] * (a + b + c)).sum(axis=0) / (24.0 * volume)


def make_particle(pid: int, vertices, triangles, epsilon: float, st: ParticleState,
                  fanout: int = 4, tree=None) -> Particle:
    """Recentre the mesh on its mass centre and build its surrogate tree
    (body.py:56-85).  `tree` may be supplied to reuse a cached build."""
    from .treebuild import build_surrogate_tree

    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles, dtype=np.int64)
    centred = v - centre_of_mass(v, t)
    if tree is None:
        corners = np.stack([centred[t[:, 0]], centred[t[:, 1]], centred[t[:, 2]]], axis=1)
        tree = build_surrogate_tree(corners, epsilon, fanout=fanout)
    radius = float(np.linalg.norm(centred, axis=1).max()) + epsilon
    return Particle(pid=pid, tree=tree, epsilon=float(epsilon), radius=radius,
                    timeline=timeline(st))


def bounding_sphere(vertices, epsilon: float) -> BoundingSphere:
    """Near-minimal sphere around the vertices plus the halo (mesh.py:335-352):
    from the box centre, 256 shrinking steps toward the farthest vertex."""
    v = np.asarray(vertices, dtype=np.float64)
    center = 0.5 * (v.min(axis=0) + v.max(axis=0))
    for k in range(256):
        delta = v - center
        far = int(np.argmax(np.einsum("ij,ij->i", delta, delta)))
        center = center + delta[far] / (k + 2.0)
    radius = float(np.linalg.norm(v - center, axis=1).max()) + epsilon
    return BoundingSphere(center=center, radius=radius)


def make_static(sid: int, vertices, triangles, epsilon: float, fanout: int = 4) -> StaticBody:
    from .treebuild import build_surrogate_tree

    if sid >= 0:
        raise ValueError(f"static ids are negative, got {sid}")
    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles, dtype=np.int64)
    corners = np.stack([v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]], axis=1)
    return StaticBody(sid=sid, tree=build_surrogate_tree(corners, epsilon, fanout=fanout),
                      epsilon=float(epsilon), sphere=bounding_sphere(v, epsilon))
