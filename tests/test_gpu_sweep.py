"""The batched per-sweep driver against the
reference engine's own sweeps.

tests/golden/engine_sweeps.npz records `ltsdem.engine.step` (engine.py:
146-261) on its "stacks" scenario: per sweep every cluster, its cache-key
fields, whether the engine computed it or reused its cached outcome
(engine.py:175-182), the result the engine used, and the particle states.
The replay feeds each sweep's clusters to `sweep.SweepDriver`, which must
(a) compute exactly the clusters the engine computed -- one batched launch
per sweep -- and (b) return the engine's results: bit for bit where no
member spins, within the SURVEY §8(c) tolerances otherwise."""

from types import SimpleNamespace

import numpy as np
import pytest

from helpers import compare_contacts, golden
from golden import scene_codec as SC

pytestmark = pytest.mark.gpu

TAU_TOL = 1e-9


@pytest.fixture(scope="module")
def S():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_15417_b200 import sweep

    return sweep


def _contacts_of(sw, i):
    lo, hi = int(sw["contacts_off"][i]), int(sw["contacts_off"][i + 1])
    return {k: v[lo:hi] for k, v in sw["contacts"].items()}


def test_engine_sweeps_replayed(S):
    from paper_2309_15417_b200 import bodies as B

    G = golden("engine_sweeps")
    particles = {}
    for rec in G["bodies"]:
        b = SC.decode_body(rec)
        particles[b.pid] = b
    statics = {}
    for rec in G["statics"]:
        s = SC.decode_body(rec)
        statics[s.sid] = s
    driver = S.SweepDriver()
    n_exact = n_tol = n_reused = 0
    for k, sw in enumerate(G["sweeps"]):
        for j, pid in enumerate(sw["ids"]):
            tl = particles[int(pid)].timeline
            tl.current = B.state(sw["position"][j], sw["velocity"][j], sw["rotation"][j],
                                 sw["angular_velocity"][j], sw["t"][j])
            tl.version = int(sw["version"][j])
        n = len(sw["dt"])
        clusters = []
        for i in range(n):
            m = tuple(int(x) for x in sw["members"][sw["members_off"][i]:sw["members_off"][i + 1]])
            st = tuple(int(x) for x in sw["statics"][sw["statics_off"][i]:sw["statics_off"][i + 1]])
            clusters.append(SimpleNamespace(members=m, t_current=float(sw["t_current"][i]), dt=float(sw["dt"][i]),
                                            statics=st))
        asked = []

        def pairs_of(i):
            asked.append(i)
            p = sw["pairs"][sw["pairs_off"][i]:sw["pairs_off"][i + 1]]
            return [(int(a), int(b)) for a, b in p]

        out = driver.results(clusters, particles, statics, pairs_of)
        want_computed = [i for i in range(n) if sw["computed"][i]]
        assert sorted(asked) == want_computed, f"sweep {k}: computed {sorted(asked)} vs engine {want_computed}"
        assert driver.last.launches == (1 if want_computed else 0)
        n_reused += n - len(want_computed)
        for i, res in enumerate(out):
            label = f"sweep {k} cluster {i}"
            spin = any(np.any(particles[m].timeline.current.angular_velocity != 0.0) for m in clusters[i].members)
            want_first = None if np.isnan(sw["res_first"][i]) else float(sw["res_first"][i])
            assert res.collision == bool(sw["res_collision"][i]), label
            assert res.narrowing_iters == int(sw["res_narrowing"][i]), label
            want_c = _contacts_of(sw, i)
            if not spin:
                n_exact += 1
                assert res.dt == float(sw["res_dt"][i]), label
                assert res.first_contact == want_first, label
                compare_contacts(res.contacts, want_c, label=label)
            else:
                n_tol += 1
                assert abs(res.dt - float(sw["res_dt"][i])) <= TAU_TOL, label
                if want_first is not None:
                    assert abs(res.first_contact - want_first) <= TAU_TOL, label
                got_c = SC.encode_contacts(res.contacts)
                for f in ("tri_a", "tri_b"):
                    got_c[f] = want_c[f]
                compare_contacts(got_c, want_c, rtol=1e-9, atol=TAU_TOL, label=label)
    assert n_reused > 0 and n_exact > 0
    print(f"{n_exact} clusters bit-exact, {n_tol} within tolerance (spinning), {n_reused} reused from the cache")
