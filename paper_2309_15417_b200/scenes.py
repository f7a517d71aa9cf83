"""Seeded synthetic workloads for the five BASELINE.json configurations.

No dataset is involved: BASELINE.json describes each configuration by its
shapes, sizes and value distributions, and these generators reproduce
them with `np.random.default_rng(230915417 + config_index)` (SURVEY.md
§8(d)).  Every generator takes a scale argument so tests can build the
same distribution at small size.  Building bodies (mass centre, recentring)
is host setup; their surrogate trees come from the GPU builder (treebuild.py).
Scene setup is not timed by `bench.py`.

c1  static pairs of 3x-subdivided noisy icospheres (1280 tris), eps 0.01
c2  dominoes: 12-tri boxes 0.1 x 0.5 x 1.0 in a row, gap 0.08, tilts, eps 1e-3
c3  granular heap: convex rocks (~124 tris), log-uniform radii, phi ~ 0.55, eps 0.005
c4  moving pairs of noisy icospheres, v ~ N(0,1), w ~ N(0,2), gap U(0,0.5), dt 0.1, eps 1e-3
c5  polydisperse mixed meshes (12 .. 20480 tris), clusters of a swept-sphere graph, eps 1e-3
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import bodies as B

SEED = 230915417

# ---------------------------------------------------------------- meshes

def icosphere(subdivisions: int):
    """Unit icosphere: 20 * 4**s triangles, outward winding."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v = v / np.linalg.norm(v, axis=1, keepdims=True)
    for _ in range(subdivisions):
        edges = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
        uniq, inv = np.unique(edges, axis=0, return_inverse=True)
        mid = v[uniq[:, 0]] + v[uniq[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        base = len(v)
        v = np.concatenate([v, mid])
        m = inv.reshape(3, -1).T + base          # midpoints of (01, 12, 20)
        f = np.concatenate([
            np.stack([f[:, 0], m[:, 0], m[:, 2]], 1),
            np.stack([f[:, 1], m[:, 1], m[:, 0]], 1),
            np.stack([f[:, 2], m[:, 2], m[:, 1]], 1),
            np.stack([m[:, 0], m[:, 1], m[:, 2]], 1)])
    return v, f


def box(dims):
    """Axis-aligned box centred at the origin, 12 triangles (mesh.py:71-93 layout)."""
    signs = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                      [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)
    tris = np.array([[0, 2, 1], [0, 3, 2], [4, 5, 6], [4, 6, 7], [0, 1, 5], [0, 5, 4],
                     [2, 3, 7], [2, 7, 6], [1, 2, 6], [1, 6, 5], [3, 0, 4], [3, 4, 7]],
                    dtype=np.int64)
    return 0.5 * signs * np.asarray(dims, dtype=np.float64), tris


def rock(rng, n_points: int = 64):
    """Convex hull of Gaussian directions projected on the unit sphere."""
    from scipy.spatial import ConvexHull

    p = rng.normal(size=(n_points, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    hull = ConvexHull(p)
    used = np.unique(hull.simplices)
    remap = -np.ones(n_points, dtype=np.int64)
    remap[used] = np.arange(len(used))
    v = p[used]
    f = remap[hull.simplices]
    a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    inward = np.einsum("ij,ij->i", np.cross(b - a, c - a), a + b + c) < 0.0
    f[inward] = f[inward][:, [0, 2, 1]]
    return v, f


def random_quaternions(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def unit_vectors(rng, n):
    d = rng.normal(size=(n, 3))
    return d / np.linalg.norm(d, axis=1, keepdims=True)


# ---------------------------------------------------------------- scenes

@dataclass
class Scene:
    """A batch of narrow-phase problems over one set of bodies.

    `pairs` are (body id a, body id b); `problem` maps each pair to a problem
    index; `dt[p]`, `t_base[p]` per problem.  Pair-mode problems (one pair
    each, like `pair_earliest_contact`) have t_base 0; cluster-mode problems
    (`compute_effective_dt`) share one bound across their pairs.
    """
    name: str
    particles: dict
    statics: dict
    pairs: list
    problem: np.ndarray
    dt: np.ndarray
    t_base: np.ndarray
    mode: str = "pair"
    meta: dict = field(default_factory=dict)

    @property
    def n_problems(self) -> int:
        return len(self.dt)

    def body(self, bid):
        return self.particles[bid] if bid >= 0 else self.statics[bid]


def _pair_scene(name, particles, pairs, dt, meta):
    n = len(pairs)
    return Scene(name=name, particles=particles, statics={}, pairs=pairs,
                 problem=np.arange(n), dt=np.full(n, float(dt)), t_base=np.zeros(n),
                 mode="pair", meta=meta)


def _noisy_icosphere_trees(rng, n, subdiv, noise, eps, radius=1.0):
    v0, f = icosphere(subdiv)
    out = []
    for _ in range(n):
        scale = radius * (1.0 + rng.uniform(-noise, noise, size=len(v0)))
        out.append((v0 * scale[:, None], f))
    return out


# The surrogate trees of a scene: `TREE_BUILDER(corners_list, epsilons)` ->
# list of SurrogateTree.  None selects the product builder, the GPU
# (`treebuild.build_surrogate_trees`, one device call for all meshes).
# CPU-only test runs install the CPU oracle's builder here (tests/conftest.py);
# both give bit-identical trees (tests/test_gpu_treebuild.py).
TREE_BUILDER = None


def build_trees(corners_list, eps) -> list:
    if TREE_BUILDER is not None:
        return TREE_BUILDER(corners_list, eps)
    from .treebuild import build_surrogate_trees

    out = []
    # bounded device batches: ~2M fine triangles per call
    lo = 0
    eps = np.broadcast_to(np.asarray(eps, dtype=np.float64), (len(corners_list),))
    while lo < len(corners_list):
        hi, tris = lo, 0
        while hi < len(corners_list) and (hi == lo or tris + len(corners_list[hi]) <= (1 << 21)):
            tris += len(corners_list[hi])
            hi += 1
        out += build_surrogate_trees(corners_list[lo:hi], eps[lo:hi])
        lo = hi
    return out


def _recentre(meshes, eps):
    """Mass centres, recentred corners (P, n, 3, 3) and bounding radii of
    meshes sharing one triangle topology, vectorised across meshes."""
    f = meshes[0][1]
    V = np.stack([np.asarray(v, dtype=np.float64) for v, _ in meshes])
    a, b, c = V[:, f[:, 0]], V[:, f[:, 1]], V[:, f[:, 2]]
    dets = np.einsum("pij,pij->pi", a, np.cross(b, c))
    vol = dets.sum(axis=1) / 6.0
    com = (dets[..., None] * (a + b + c)).sum(axis=1) / (24.0 * vol)[:, None]
    Vc = V - com[:, None, :]
    corners = np.stack([Vc[:, f[:, 0]], Vc[:, f[:, 1]], Vc[:, f[:, 2]]], axis=2)
    radius = np.linalg.norm(Vc, axis=2).max(axis=1) + eps
    return corners, radius


def make_particles(ids, meshes, eps, states, workers=None):
    """Batched make_particle for meshes sharing one triangle topology:
    centres of mass and recentring vectorised across particles, all trees
    in one builder call."""
    corners, radius = _recentre(meshes, eps)
    trees = build_trees(list(corners), eps)
    return [B.Particle(pid=int(i), tree=t, epsilon=float(eps), radius=float(r), timeline=B.timeline(st))
            for i, t, r, st in zip(ids, trees, radius, states)]


def make_particles_each(specs, workers=None, share=None):
    """B.make_particle for every (pid, vertices, faces, eps, state, key) of
    `specs` (meshes of any topology), all trees in one builder call.  Specs
    with an equal non-None `key` share the tree of the first one (identical
    meshes).  Same particles as the serial loop."""
    first = {}
    todo = []
    for sp in specs:
        key = sp[5]
        if key is None or key not in first:
            if key is not None:
                first[key] = sp[0]
            todo.append(sp)
    corners = []
    for pid, v, f, eps, st, key in todo:
        v = np.asarray(v, dtype=np.float64)
        f = np.asarray(f, dtype=np.int64)
        c = v - B.centre_of_mass(v, f)
        corners.append(np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1))
    trees = build_trees(corners, [sp[3] for sp in todo])
    tree_of = {sp[0]: t for sp, t in zip(todo, trees)}
    out = {}
    for pid, v, f, eps, st, key in specs:
        tree = tree_of[pid] if pid in tree_of else tree_of[first[key]]
        out[pid] = B.make_particle(pid, v, f, eps, st, tree=tree)
    return out


def config1(n_pairs: int = 1024, subdiv: int = 3, seed_offset: int = 1) -> Scene:
    """c1: static noisy-icosphere pairs, centre distance U(1.9, 2.1), eps 0.01."""
    rng = np.random.default_rng(SEED + seed_offset)
    eps = 0.01
    meshes = _noisy_icosphere_trees(rng, 2 * n_pairs, subdiv, 0.05, eps)
    quats = random_quaternions(rng, 2 * n_pairs)
    dist = rng.uniform(1.9, 2.1, size=n_pairs)
    axes = unit_vectors(rng, n_pairs)
    states = [B.state((1.0 if pid % 2 else -1.0) * 0.5 * dist[pid // 2] * axes[pid // 2], rotation=quats[pid])
              for pid in range(2 * n_pairs)]
    made = make_particles(range(2 * n_pairs), meshes, eps, states)
    particles = {p.pid: p for p in made}
    pairs = [(2 * k, 2 * k + 1) for k in range(n_pairs)]
    return _pair_scene("c1", particles, pairs, 0.0,
                       {"eps": eps, "tris": 20 * 4 ** subdiv, "n_pairs": n_pairs})


def config2(n_boxes: int = 4096, seed_offset: int = 2) -> Scene:
    """c2: dominoes 0.1 x 0.5 x 1.0, face gap 0.08 (pitch 0.18), tilt about y."""
    rng = np.random.default_rng(SEED + seed_offset)
    eps = 1e-3
    v, f = box((0.1, 0.5, 1.0))
    tilt = rng.uniform(0.0, 0.3, size=n_boxes)
    particles = {}
    c = v - B.centre_of_mass(v, f)
    tree = build_trees([np.stack([c[f[:, 0]], c[f[:, 1]], c[f[:, 2]]], axis=1)], eps)[0]
    for i in range(n_boxes):
        q = np.array([np.cos(0.5 * tilt[i]), 0.0, np.sin(0.5 * tilt[i]), 0.0])
        st = B.state((0.18 * i, 0.0, 0.5), rotation=q)
        particles[i] = B.make_particle(i, v, f, eps, st, tree=tree)
    r = particles[0].radius
    pairs = []
    for i in range(n_boxes):
        for j in range(i + 1, n_boxes):
            if 0.18 * (j - i) > 2 * r:
                break
            pairs.append((i, j))
    return _pair_scene("c2", particles, pairs, 0.0, {"eps": eps, "n_boxes": n_boxes})


def _relax(rng, radii, phi, overlap=0.02, iters=200):
    """Grow-and-relax a polydisperse sphere packing at volume fraction phi."""
    from scipy.spatial import cKDTree

    n = len(radii)
    vol = (4.0 / 3.0) * np.pi * (radii ** 3).sum() / phi
    side = vol ** (1.0 / 3.0)
    x = rng.uniform(0.0, side, size=(n, 3))
    rmax = radii.max()
    for _ in range(iters):
        tree = cKDTree(x, boxsize=side)
        ij = tree.query_pairs(2.0 * rmax, output_type="ndarray")
        d = x[ij[:, 1]] - x[ij[:, 0]]
        d -= side * np.round(d / side)
        dist = np.linalg.norm(d, axis=1)
        target = (radii[ij[:, 0]] + radii[ij[:, 1]]) * (1.0 - overlap)
        push = np.maximum(target - dist, 0.0)
        if not (push > 1e-9).any():
            break
        u = d / np.maximum(dist, 1e-12)[:, None]
        delta = np.zeros_like(x)
        np.add.at(delta, ij[:, 0], -0.5 * push[:, None] * u)
        np.add.at(delta, ij[:, 1], 0.5 * push[:, None] * u)
        x = np.mod(x + delta, side)
    return x, side


def config3(n_rocks: int = 20000, phi: float = 0.55, seed_offset: int = 3) -> Scene:
    """c3: convex rocks with log-uniform radii 0.5..5 packed at phi ~ 0.55."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(SEED + seed_offset)
    eps = 0.005
    radii = np.exp(rng.uniform(np.log(0.5), np.log(5.0), size=n_rocks))
    specs = []
    for i in range(n_rocks):
        v, f = rock(rng)
        q = random_quaternions(rng, 1)[0]
        specs.append((i, v * radii[i], f, eps, B.state(np.zeros(3), rotation=q), None))
    particles = make_particles_each(specs)
    bound = np.array([particles[i].radius for i in range(n_rocks)])
    x, side = _relax(rng, bound, phi)
    for i in range(n_rocks):
        particles[i].timeline.current.position = x[i].copy()
        particles[i].timeline.old.position = x[i].copy()
    tree = cKDTree(x)
    ij = tree.query_pairs(2.0 * bound.max(), output_type="ndarray")
    d = np.linalg.norm(x[ij[:, 0]] - x[ij[:, 1]], axis=1)
    keep = d <= bound[ij[:, 0]] + bound[ij[:, 1]]
    ij = ij[keep]
    ij = ij[np.lexsort((ij[:, 1], ij[:, 0]))]
    pairs = [(int(a), int(b)) for a, b in ij]
    achieved = (4.0 / 3.0) * np.pi * (bound ** 3).sum() / side ** 3
    return _pair_scene("c3", particles, pairs, 0.0,
                       {"eps": eps, "n_rocks": n_rocks, "phi_bounding": float(achieved)})


def config4_raw(n_pairs: int = 8192, subdiv: int = 3, dt: float = 0.1, seed_offset: int = 4) -> dict:
    """c4's seeded draws without building trees: per body its mesh (not yet
    recentred), bounding radius and snapshot state (positions set), so a
    fixture generator can rebuild chosen pairs of the bench workload with
    the reference's own make_particle."""
    rng = np.random.default_rng(SEED + seed_offset)
    eps = 1e-3
    meshes = _noisy_icosphere_trees(rng, 2 * n_pairs, subdiv, 0.05, eps)
    quats = random_quaternions(rng, 2 * n_pairs)
    vel = rng.normal(0.0, 1.0, size=(2 * n_pairs, 3))
    spin = rng.normal(0.0, 2.0, size=(2 * n_pairs, 3))
    gaps = rng.uniform(0.0, 0.5, size=n_pairs)
    axes = unit_vectors(rng, n_pairs)
    _, radius = _recentre(meshes, eps)
    states = []
    for pid in range(2 * n_pairs):
        k = pid // 2
        sep = radius[2 * k] + radius[2 * k + 1] + gaps[k]
        pos = (0.5 if pid % 2 else -0.5) * sep * axes[k]
        states.append(B.state(pos, velocity=vel[pid], rotation=quats[pid], angular_velocity=spin[pid]))
    return {"eps": eps, "dt": dt, "meshes": meshes, "radius": radius, "states": states,
            "pairs": [(2 * k, 2 * k + 1) for k in range(n_pairs)], "gaps": gaps, "axes": axes}


def config4(n_pairs: int = 8192, subdiv: int = 3, dt: float = 0.1, seed_offset: int = 4) -> Scene:
    """c4: moving icosphere pairs, v ~ N(0,1)^3, w ~ N(0,2)^3, gap U(0,0.5)."""
    raw = config4_raw(n_pairs, subdiv, dt, seed_offset)
    made = make_particles(range(2 * n_pairs), raw["meshes"], raw["eps"], raw["states"])
    particles = {p.pid: p for p in made}
    return _pair_scene("c4", particles, raw["pairs"], dt,
                       {"eps": raw["eps"], "tris": 20 * 4 ** subdiv, "n_pairs": n_pairs})


def config5_raw(n_particles: int = 2000, dt: float = 0.1, max_subdiv: int = 5, seed_offset: int = 5) -> dict:
    """c5's seeded draws without building trees: per particle its mesh (not
    yet recentred), kind, radius and snapshot state after the packing, the
    swept-sphere pairs and their clusters."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(SEED + seed_offset)
    eps = 1e-3
    radii = np.exp(rng.uniform(np.log(0.05), np.log(5.0), size=n_particles))
    kinds = rng.integers(0, max_subdiv + 2, size=n_particles)   # max_subdiv+1 -> box
    vel = rng.normal(0.0, 1.0, size=(n_particles, 3))
    spin = rng.normal(0.0, 1.0, size=(n_particles, 3))
    quats = random_quaternions(rng, n_particles)
    meshes = []
    bound = np.empty(n_particles)
    for i in range(n_particles):
        kind = int(kinds[i])
        v, f = icosphere(kind) if kind <= max_subdiv else box((1.0, 0.8, 0.6))
        v = v * radii[i]
        meshes.append((v, f))
        bound[i] = float(np.linalg.norm(v - B.centre_of_mass(v, f), axis=1).max()) + eps  # make_particle's radius
    x, _ = _relax(rng, bound, 0.35, overlap=-0.002)
    states = [B.state(x[i].copy(), velocity=vel[i], rotation=quats[i], angular_velocity=spin[i])
              for i in range(n_particles)]
    # swept bounding spheres over [0, dt]
    reach = bound + dt * np.linalg.norm(vel, axis=1)
    tree = cKDTree(x)
    ij = tree.query_pairs(2.0 * reach.max(), output_type="ndarray")
    d = np.linalg.norm(x[ij[:, 0]] - x[ij[:, 1]], axis=1)
    ij = ij[d <= reach[ij[:, 0]] + reach[ij[:, 1]]]
    ij = ij[np.lexsort((ij[:, 1], ij[:, 0]))]
    graph = coo_matrix((np.ones(len(ij)), (ij[:, 0], ij[:, 1])), shape=(n_particles,) * 2)
    _, label = connected_components(graph, directed=False)
    pairs = [(int(a), int(b)) for a, b in ij]
    comp = label[ij[:, 0]] if len(ij) else np.zeros(0, dtype=np.int64)
    uniq, problem = np.unique(comp, return_inverse=True)
    return {"eps": eps, "dt": dt, "meshes": meshes, "kinds": kinds, "radii": radii, "radius": bound,
            "states": states, "pairs": pairs, "problem": np.asarray(problem, dtype=np.int64),
            "n_problems": len(uniq)}


def config5(n_particles: int = 2000, dt: float = 0.1, max_subdiv: int = 5,
            seed_offset: int = 5) -> Scene:
    """c5: polydisperse icospheres (20..20480 tris) and boxes, size ratio
    100:1, non-overlapping packing, clusters of the swept-sphere graph."""
    raw = config5_raw(n_particles, dt, max_subdiv, seed_offset)
    eps = raw["eps"]
    particles = make_particles_each(
        [(i, raw["meshes"][i][0], raw["meshes"][i][1], eps, raw["states"][i],
          (int(raw["kinds"][i]), float(raw["radii"][i]))) for i in range(n_particles)])
    n_prob = raw["n_problems"]
    return Scene(name="c5", particles=particles, statics={}, pairs=raw["pairs"],
                 problem=raw["problem"], dt=np.full(n_prob, float(dt)),
                 t_base=np.zeros(n_prob), mode="cluster",
                 meta={"eps": eps, "n_particles": n_particles, "clusters": n_prob})


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}
