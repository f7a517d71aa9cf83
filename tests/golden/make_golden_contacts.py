"""Generate the contact-consumer golden fixtures by running the REFERENCE itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_contacts.py

Output (committed): tests/golden/contacts.npz, a list of cases.  Each case
is one cluster: body records (the layout of include/ltsgpu.h,
ltsg_solve_input), its contact list, the solver configuration, and the
reference's outputs:

* `ltsdem.contacts.solve_impulses` (contacts.py:114-198): velocities and
  angular velocities in the solution dict's order, iterations, converged,
  normal and friction impulses, and `color_contact_graph` (:58-78);
* `integrate_cluster` (:225-253) followed by `apply_separation` (:256-285):
  every member's new snapshot.

Cases: the reference's own test_contacts.py scenarios, and seeded random
clusters (cube particles made by the reference's make_particle, random
states, contacts on random body pairs and statics), non-spinning (bit-exact
on the GPU) and spinning (quaternions.advance's sin/cos: tolerance).
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

from ltsdem.body import initial_state, make_particle  # noqa: E402
from ltsdem.ccd import ContactPoint, NarrowResult  # noqa: E402
from ltsdem.clustering import Cluster  # noqa: E402
from ltsdem.contacts import (  # noqa: E402
    SolverConfig, apply_separation, color_contact_graph, integrate_cluster, solve_impulses,
)
from ltsdem.mesh import make_cube, make_noisy_sphere  # noqa: E402
from ltsdem.state import extrapolate_free_flight, roll_over  # noqa: E402

import gio  # noqa: E402
from paper_2309_15417_b200 import scenes as S  # noqa: E402


def body_record(p):
    s = p.timeline.current
    r = np.zeros(24)
    r[0:3], r[3:6], r[6:10], r[10:13], r[13] = s.position, s.velocity, s.rotation, s.angular_velocity, s.t
    r[14] = 1.0 / p.mass.mass
    r[15:24] = p.mass.inverse_inertia.reshape(9)
    return r


def record(name, particles, contacts, cfg, t_current, dt, spin=False):
    ids = sorted(particles)
    sol = solve_impulses(contacts, particles, cfg)
    classes = color_contact_graph(contacts)
    members = tuple(sorted({b for c in contacts for b in (c.body_a, c.body_b) if b >= 0} | set(ids)))
    cluster = Cluster(members=members, t_current=t_current, dt=dt)
    result = NarrowResult(dt=dt, contacts=contacts, narrowing_iters=1 if contacts else 0,
                          bound_history=[], collision=bool(contacts))
    recs = np.array([body_record(particles[i]) for i in ids])
    integrate_cluster(cluster, particles, result, sol if contacts else None)
    apply_separation(contacts, particles, cfg.beta)
    new = np.array([np.concatenate([particles[i].timeline.new.position, particles[i].timeline.new.velocity,
                                    particles[i].timeline.new.rotation,
                                    particles[i].timeline.new.angular_velocity, [particles[i].timeline.new.t]])
                    for i in ids])
    cls_of = np.zeros(len(contacts), dtype=np.int64)
    for k, cl in enumerate(classes):
        cls_of[cl] = k
    print(f"  {name}: {len(ids)} bodies, {len(contacts)} contacts, {sol.iterations} iterations, "
          f"converged {sol.converged}", flush=True)
    return {
        "name": name, "ids": np.array(ids, dtype=np.int64), "rec": recs,
        "body_a": np.array([c.body_a for c in contacts], dtype=np.int64).reshape(-1),
        "body_b": np.array([c.body_b for c in contacts], dtype=np.int64).reshape(-1),
        "position": np.array([c.position for c in contacts], dtype=np.float64).reshape(-1, 3),
        "normal": np.array([c.normal for c in contacts], dtype=np.float64).reshape(-1, 3),
        "t": np.array([c.t for c in contacts], dtype=np.float64).reshape(-1),
        "depth": np.array([c.depth for c in contacts], dtype=np.float64).reshape(-1),
        "cfg": {"restitution": cfg.restitution, "friction": cfg.friction, "relaxation": cfg.relaxation,
                "penalty": cfg.penalty, "threshold": cfg.threshold, "max_iterations": cfg.max_iterations,
                "beta": cfg.beta},
        "t_current": float(t_current), "dt": float(dt), "spin": bool(spin),
        "sol_ids": np.array(list(sol.velocities.keys()), dtype=np.int64),
        "sol_vel": np.array(list(sol.velocities.values()), dtype=np.float64).reshape(-1, 3),
        "sol_ang": np.array(list(sol.angular_velocities.values()), dtype=np.float64).reshape(-1, 3),
        "iterations": int(sol.iterations), "converged": bool(sol.converged),
        "lam": np.array(sol.normal_impulses, dtype=np.float64),
        "fric": np.array(sol.friction_impulses, dtype=np.float64).reshape(-1, 3),
        "color": cls_of, "new": new,
    }


def cube(pid, position, velocity=(0.0, 0.0, 0.0), omega=(0.0, 0.0, 0.0), edge=1.0, rotation=None):
    return make_particle(pid, make_cube(np.zeros(3), edge), epsilon=0.01,
                         state=initial_state(np.array(position, dtype=float), velocity=np.array(velocity, dtype=float),
                                             rotation=rotation, angular_velocity=np.array(omega, dtype=float)))


def contact(a, b, position, normal, t=0.0, depth=0.0):
    return ContactPoint(body_a=a, body_b=b, position=np.array(position, dtype=float),
                        normal=np.array(normal, dtype=float), depth=depth, t=t, threshold=0.02)


TIGHT = SolverConfig(threshold=1e-11)


def reference_scenarios():
    out = []
    a = cube(0, (-0.51, 0, 0), velocity=(1, 0, 0))
    b = cube(1, (0.51, 0, 0), velocity=(-1, 0, 0))
    out.append(record("head_on", {0: a, 1: b}, [contact(0, 1, (0, 0, 0), (-1, 0, 0))], TIGHT, 0.0, 0.5))
    a = cube(0, (-0.51, 0, 0), velocity=(1, 0, 0))
    b = cube(1, (0.51, 0, 0), velocity=(-1, 0, 0))
    out.append(record("inelastic", {0: a, 1: b}, [contact(0, 1, (0, 0, 0), (-1, 0, 0))],
                      SolverConfig(restitution=0.0, threshold=1e-9), 0.0, 0.5))
    a = cube(0, (0, 0, 0.5), velocity=(1, 0, -2))
    out.append(record("oblique_floor", {0: a}, [contact(0, -1, (0, 0, 0), (0, 0, 1), depth=0.004)], TIGHT, 0.0, 0.2))
    left = cube(0, (-1.02, 0, 0), velocity=(1, 0, 0))
    mid = cube(1, (0, 0, 0))
    right = cube(2, (1.02, 0, 0), velocity=(-1, 0, 0))
    out.append(record("two_impacts", {0: left, 1: mid, 2: right},
                      [contact(1, 0, (-0.51, 0, 0), (1, 0, 0)), contact(1, 2, (0.51, 0, 0), (-1, 0, 0))],
                      TIGHT, 0.0, 0.3))
    a = cube(0, (0, 0, 0), velocity=(1, 0, 0))
    b = cube(1, (3, 0, 0), velocity=(-1, 0, 0))
    out.append(record("late_contact", {0: a, 1: b}, [contact(0, 1, (1.5, 0, 0), (-1, 0, 0), t=0.4)],
                      SolverConfig(), 0.0, 1.0))
    a = cube(0, (0, 0, 0), velocity=(2, 0, 0))
    out.append(record("free_flight", {0: a}, [], SolverConfig(), 0.0, 0.5))
    return out


def random_cluster(rng, name, n_bodies, n_contacts, spin, cfg, statics=(-1, -2)):
    particles = {}
    for pid in range(n_bodies):
        mesh = make_cube(np.zeros(3), float(rng.uniform(0.4, 1.5))) if pid % 2 else \
            make_noisy_sphere(float(rng.uniform(0.3, 1.0)), 80, 1.05, int(rng.integers(1 << 30)))
        q = S.random_quaternions(rng, 1)[0]
        p = make_particle(pid, mesh, epsilon=0.01,
                          state=initial_state(rng.uniform(-2, 2, 3), velocity=rng.normal(size=3),
                                              rotation=q, angular_velocity=rng.normal(size=3) if spin else np.zeros(3),
                                              t=float(rng.choice([0.0, 0.05]))))
        if rng.uniform() < 0.3:  # a completed step: old and current differ
            p.timeline.new = extrapolate_free_flight(p.timeline.current, 0.05)
            roll_over(p.timeline)
        particles[pid] = p
    t_current = max(p.timeline.current.t for p in particles.values())
    contacts = []
    for _ in range(n_contacts):
        a = int(rng.integers(n_bodies))
        b = int(rng.choice([x for x in range(n_bodies) if x != a] + list(statics)))
        nrm = rng.normal(size=3)
        nrm /= np.linalg.norm(nrm)
        contacts.append(contact(a, b, rng.uniform(-2, 2, 3), nrm, t=t_current + float(rng.uniform(0, 0.1)),
                                depth=float(rng.choice([0.0, rng.uniform(0, 0.01)]))))
    return record(name, particles, contacts, cfg, t_current, 0.1, spin=spin)


def main():
    print("contact-consumer goldens (reference run)", flush=True)
    cases = reference_scenarios()
    rng = np.random.default_rng(2309)
    for k in range(10):
        cfg = SolverConfig(restitution=float(rng.uniform(0, 1)), friction=float(rng.choice([0.0, 0.3, 0.8])),
                           relaxation=float(rng.uniform(0.3, 1.0)), threshold=float(rng.choice([1e-4, 1e-9])),
                           max_iterations=int(rng.choice([16, 256])))
        cases.append(random_cluster(rng, f"random_{k}", int(rng.integers(2, 12)), int(rng.integers(1, 30)),
                                    spin=False, cfg=cfg))
    for k in range(4):
        cases.append(random_cluster(rng, f"spin_{k}", int(rng.integers(2, 8)), int(rng.integers(1, 12)),
                                    spin=True, cfg=SolverConfig()))
    cases.append(random_cluster(rng, "large", 60, 200, spin=False, cfg=SolverConfig(max_iterations=64)))
    gio.save(os.path.join(HERE, "contacts.npz"), {"cases": cases})
    print("wrote contacts.npz")


if __name__ == "__main__":
    main()
