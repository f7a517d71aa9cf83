"""Record whole sweeps of the REFERENCE engine, stage by stage.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_engine.py

Output (committed): tests/golden/engine_steps.npz.  `ltsdem.engine.step`
(engine.py:146-261) runs on its own "stacks" scenario with the module
globals it resolves at call time wrapped, so that every sweep records what
each stage on the GPU path saw and produced inside a real engine run:

* the particles' timelines (old and current snapshots) at the start of the
  sweep and the collision graph `build_collision_graph` returned for them
  (engine.py:157): edges in dict order with their windows, static links,
  step bounds;
* every `solve_impulses` call (engine.py:141, :215): its contacts and the
  solution it returned;
* every commit (engine.py:227-228): the cluster, the committed result, the
  solution, and each member's `timeline.new` after `integrate_cluster` and
  `apply_separation`.

tests/test_gpu_engine_steps.py replays each stage through the package's
drop-in modules (the narrow-phase stage of the same scenario is replayed by
tests/test_gpu_sweep.py from engine_sweeps.npz).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import gio  # noqa: E402
import scene_codec as SC  # noqa: E402


def _states(parts, ids, which):
    st = [getattr(parts[p].timeline, which) for p in ids]
    return {"position": np.array([s.position for s in st]), "velocity": np.array([s.velocity for s in st]),
            "rotation": np.array([s.rotation for s in st]),
            "angular_velocity": np.array([s.angular_velocity for s in st]), "t": np.array([s.t for s in st])}


def main(n_sweeps=40):
    from ltsdem import engine
    from ltsdem.scenarios import ScenarioConfig, build_world

    world = build_world(ScenarioConfig("stacks", rows=1, seed=3))
    parts = world.particles
    ids = sorted(parts)
    sweeps = []
    cur = {}
    f_graph, f_solve, f_int, f_sep = (engine.build_collision_graph, engine.solve_impulses,
                                      engine.integrate_cluster, engine.apply_separation)

    def graph(particles, statics, policy, *a, **kw):
        cur.clear()
        cur.update({"old": _states(parts, ids, "old"), "current": _states(parts, ids, "current"),
                    "solves": [], "commits": []})
        g = f_graph(particles, statics, policy, *a, **kw)
        keys = list(g.edges)
        links = [(p, s) for p, ss in g.static_links.items() for s in ss]
        cur["graph"] = {"edges": np.array(keys, dtype=np.int64).reshape(-1, 2),
                        "windows": np.array([g.edges[k] for k in keys], dtype=np.float64).reshape(-1, 2),
                        "links": np.array(links, dtype=np.int64).reshape(-1, 2),
                        "link_order": np.array(list(g.static_links), dtype=np.int64),
                        "dts": np.array([g.dts[p] for p in ids])}
        return g

    def solve(contacts, particles, config=None):
        sol = f_solve(contacts, particles, config)
        bids = list(sol.velocities)
        cur["solves"].append({
            "contacts": SC.encode_contacts(list(contacts)),
            "bodies": np.array(bids, dtype=np.int64),
            "velocity": np.array([sol.velocities[b] for b in bids]).reshape(-1, 3),
            "angular_velocity": np.array([sol.angular_velocities[b] for b in bids]).reshape(-1, 3),
            "iterations": np.int64(sol.iterations), "converged": np.bool_(sol.converged)})
        return sol

    pending = {}

    def integrate(cluster, particles, result, solution):
        pending["c"] = (cluster, result, solution)
        return f_int(cluster, particles, result, solution)

    def separate(contacts, particles, beta):
        out = f_sep(contacts, particles, beta)
        cluster, result, solution = pending.pop("c")
        mem = list(cluster.members)
        bids = list(solution.velocities) if solution is not None else []
        new = [parts[p].timeline.new for p in mem]
        cur["commits"].append({
            "members": np.array(mem, dtype=np.int64), "t_current": np.float64(cluster.t_current),
            "dt": np.float64(result.dt), "contacts": SC.encode_contacts(list(result.contacts)),
            "has_solution": np.bool_(solution is not None),
            "sol_bodies": np.array(bids, dtype=np.int64),
            "sol_velocity": np.array([solution.velocities[b] for b in bids]).reshape(-1, 3),
            "sol_angular_velocity": np.array([solution.angular_velocities[b] for b in bids]).reshape(-1, 3),
            "beta": np.float64(beta),
            "new": {"position": np.array([s.position for s in new]), "velocity": np.array([s.velocity for s in new]),
                    "rotation": np.array([s.rotation for s in new]),
                    "angular_velocity": np.array([s.angular_velocity for s in new]),
                    "t": np.array([s.t for s in new])}})
        return out

    engine.build_collision_graph, engine.solve_impulses = graph, solve
    engine.integrate_cluster, engine.apply_separation = integrate, separate
    bodies0 = [SC.encode_body(parts[p]) for p in ids]
    assert all(np.all(parts[p].sphere.center == 0.0) for p in ids)  # make_particle pins it (body.py:73-76)
    spheres = {"radius": np.array([parts[p].sphere.radius for p in ids]),
               "static_center": np.array([s.sphere.center for s in world.statics.values()]).reshape(-1, 3),
               "static_radius": np.array([s.sphere.radius for s in world.statics.values()])}
    mass = {"inv_mass": np.array([1.0 / parts[p].mass.mass for p in ids]),
            "inv_inertia": np.array([parts[p].mass.inverse_inertia for p in ids]).reshape(-1, 3, 3)}
    try:
        for _ in range(n_sweeps):
            engine.step(world)
            sweeps.append({k: (dict(v) if isinstance(v, dict) else list(v)) for k, v in cur.items()})
    finally:
        engine.build_collision_graph, engine.solve_impulses = f_graph, f_solve
        engine.integrate_cluster, engine.apply_separation = f_int, f_sep
    cfg = world.config
    out = {"ids": np.array(ids, dtype=np.int64), "bodies": bodies0, "mass": mass, "spheres": spheres,
           "statics": [SC.encode_body(s) for s in world.statics.values()],
           "policy": {"dt_max": np.float64(cfg.policy.dt_max), "growth": np.float64(cfg.policy.growth)},
           "solver": {k: np.float64(getattr(cfg.solver, k)) for k in
                      ("restitution", "friction", "relaxation", "penalty", "threshold", "max_iterations", "beta")},
           "sweeps": sweeps}
    n_edges = sum(len(s["graph"]["edges"]) for s in sweeps)
    n_solves = sum(len(s["solves"]) for s in sweeps)
    n_commits = sum(len(s["commits"]) for s in sweeps)
    n_spin = sum(int(np.any(s["current"]["angular_velocity"] != 0.0)) for s in sweeps)
    path = os.path.join(HERE, "engine_steps.npz")
    gio.save(path, out)
    print(f"engine steps: {len(sweeps)} sweeps, {len(ids)} particles, {n_edges} edges, {n_solves} solves, "
          f"{n_commits} commits, {n_spin} sweeps with spin; {os.path.getsize(path) / 1e3:.0f} kB", flush=True)


if __name__ == "__main__":
    main()
