"""The CPU oracle against the reference's own outputs (golden fixtures).

Every fixture was produced by running the reference (`ltsdem`) itself
(tests/golden/make_golden.py).  The oracle must reproduce it bit for bit:
the same floating-point operations in the same order.  This pins the
oracle before anything is checked against it.
"""

import numpy as np
import pytest

from helpers import compare_contacts, compare_result, golden, run_case
from oracle import narrow_oracle as O


def test_point_triangle_rows_bit_exact():
    g = golden("kernels")["pt"]
    d, c, _ = O.point_triangle(g["p"], g["a"], g["b"], g["c"])
    np.testing.assert_array_equal(d, g["dist"])
    np.testing.assert_array_equal(c, g["closest"])


def test_segment_segment_rows_bit_exact():
    g = golden("kernels")["ss"]
    d, c1, c2 = O.segment_segment(g["p1"], g["q1"], g["p2"], g["q2"])
    np.testing.assert_array_equal(d, g["dist"])
    np.testing.assert_array_equal(c1, g["c1"])
    np.testing.assert_array_equal(c2, g["c2"])


def test_feature_distance_rows_bit_exact():
    g = golden("kernels")["feat"]
    np.testing.assert_array_equal(O.tri_pair_distance(g["ta"], g["tb"]), g["dist"])


def test_witness_points_and_normals_bit_exact():
    g = golden("witness")
    for i in range(len(g["ta"])):
        d, pa, pb = O.tri_pair_witness(g["ta"][i], g["tb"][i])
        assert d == g["dist"][i]
        np.testing.assert_array_equal(pa, g["pa"][i])
        np.testing.assert_array_equal(pb, g["pb"][i])
        np.testing.assert_array_equal(O.unit_face_normal(g["ta"][i]), g["na"][i])
        np.testing.assert_array_equal(O.unit_face_normal(g["tb"][i]), g["nb"][i])


def test_overlap_centroid_bit_exact():
    g = golden("witness")
    for i in range(len(g["ov_a"])):
        n = O.unit_face_normal(g["ov_a"][i])
        out = O.overlap_centroid(g["ov_a"][i], g["ov_b"][i], n)
        assert (out is not None) == g["ov_has"][i]
        if out is not None:
            np.testing.assert_array_equal(out, g["ov_centroid"][i])


def _contacts(soa):
    return [O.Contact(int(soa["body_a"][i]), int(soa["body_b"][i]), soa["position"][i].copy(),
                      soa["normal"][i].copy(), float(soa["depth"][i]), float(soa["t"][i]),
                      int(soa["tri_a"][i]), int(soa["tri_b"][i]), float(soa["threshold"][i]))
            for i in range(len(soa["t"]))]


def test_fusion_bit_exact():
    for k, case in enumerate(golden("fusion")["cases"]):
        compare_contacts(O.fuse(_contacts(case["raw"])), case["fused"], label=f"fusion {k}")


def _scene_ids(name):
    return [c["name"] for c in golden(name)["cases"]]


@pytest.mark.parametrize("idx", range(len(golden("scenes_ccd")["cases"])),
                         ids=_scene_ids("scenes_ccd"))
def test_reference_test_scenes_bit_exact(idx):
    case = golden("scenes_ccd")["cases"][idx]
    res = run_case(O, case)
    compare_result(res, case["result"], raw=res.raw, label=case["name"])
    assert sum(res.stats.values()) == case["rows"]


@pytest.mark.parametrize("idx", range(len(golden("scenes_configs")["cases"])),
                         ids=_scene_ids("scenes_configs"))
def test_config_shaped_scenes_bit_exact(idx):
    case = golden("scenes_configs")["cases"][idx]
    res = run_case(O, case)
    compare_result(res, case["result"], raw=res.raw, label=case["name"])
    assert sum(res.stats.values()) == case["rows"]


def test_acceptance_criterion2_pairs_bit_exact():
    """The 200 seeded pairs of the reference's acceptance criterion 2
    (test_acceptance.py:280-353), replayed; exhaustive mode on the first 30."""
    for case in golden("scenes_crit2")["cases"]:
        res = run_case(O, case)
        compare_result(res, case["result"], raw=res.raw, label=case["name"])
        assert sum(res.stats.values()) == case["rows"], case["name"]
        if "exhaustive_result" in case:
            ex = run_case(O, case, exhaustive=True)
            compare_result(ex, case["exhaustive_result"], raw=ex.raw, label=case["name"] + " ex")
            assert sum(ex.stats.values()) == case["exhaustive_rows"]


# bench-shaped scenes (c4 at 1280 triangles, c5 20480-triangle icospheres vs
# boxes): the cheapest ones keep the CPU suite within minutes; every case is
# checked against the GPU in tests/test_gpu_parity.py
_BASELINE_CPU = [c["name"] for c in golden("scenes_baseline")["cases"] if c["ref_seconds"] < 10.0][:4]


@pytest.mark.parametrize("name", _BASELINE_CPU)
def test_bench_shaped_scenes_bit_exact(name):
    case = next(c for c in golden("scenes_baseline")["cases"] if c["name"] == name)
    res = run_case(O, case)
    compare_result(res, case["result"], raw=res.raw, label=case["name"])
    assert sum(res.stats.values()) == case["rows"]


def test_bench_shaped_scenes_come_from_the_bench_workloads():
    """The fixture bodies are the bench scenes' bodies: same snapshot states
    (bit for bit) as scenes.config4_raw / config5_raw at their BASELINE sizes."""
    from paper_2309_15417_b200 import scenes

    cases = golden("scenes_baseline")["cases"]
    raws = {"c4": scenes.config4_raw(), "c5": scenes.config5_raw()}
    assert sum(c["name"].startswith("c4_") for c in cases) >= 8
    assert sum(c["name"].startswith("c5_") for c in cases) >= 2
    assert sum(c["result"]["collision"] for c in cases if c["name"].startswith("c4_")) >= 3
    for case in cases:
        raw = raws[case["name"][:2]]
        for b in case["bodies"]:
            st = raw["states"][b["id"]]
            for f in ("position", "velocity", "rotation", "angular_velocity"):
                np.testing.assert_array_equal(b[f], getattr(st, f), err_msg=f"{case['name']} body {b['id']} {f}")
        if case["name"].startswith("c5_bench_cluster"):
            sel = np.flatnonzero(raw["problem"] == case["bench_index"])
            assert [tuple(raw["pairs"][i]) for i in sel] == [tuple(p) for p in case["pairs"]]
        if case["name"].startswith("c4_"):
            assert tuple(raw["pairs"][case["bench_index"]]) == tuple(case["pairs"][0])
        sizes = [len(lv["fine_f"]) for b in case["bodies"] for lv in b["tree"][:1] if "fine_f" in lv]
        if case["name"].startswith("c4_"):
            assert sizes == [1280, 1280]
        else:
            assert 20480 in sizes


def test_engine_sweeps_pinned():
    """The oracle reproduces every result the reference engine computed in
    the recorded sweeps (tests/golden/engine_sweeps.npz), bit for bit."""
    from types import SimpleNamespace

    from golden import scene_codec as SC
    from paper_2309_15417_b200 import bodies as B

    G = golden("engine_sweeps")
    particles = {}
    for rec in G["bodies"]:
        b = SC.decode_body(rec)
        particles[b.pid] = b
    statics = {SC.decode_body(r).sid: SC.decode_body(r) for r in G["statics"]}
    checked = 0
    for sw in G["sweeps"]:
        for j, pid in enumerate(sw["ids"]):
            particles[int(pid)].timeline.current = B.state(sw["position"][j], sw["velocity"][j], sw["rotation"][j],
                                                           sw["angular_velocity"][j], sw["t"][j])
        for i in np.flatnonzero(sw["computed"]):
            cl = SimpleNamespace(t_current=float(sw["t_current"][i]), dt=float(sw["dt"][i]))
            pairs = [(int(a), int(b)) for a, b in sw["pairs"][sw["pairs_off"][i]:sw["pairs_off"][i + 1]]]
            res = O.compute_effective_dt(cl, particles, statics, pairs)
            assert res.dt == sw["res_dt"][i] and res.collision == bool(sw["res_collision"][i])
            lo, hi = int(sw["contacts_off"][i]), int(sw["contacts_off"][i + 1])
            compare_contacts(res.contacts, {k: v[lo:hi] for k, v in sw["contacts"].items()})
            checked += 1
    assert checked == sum(int(sw["computed"].sum()) for sw in G["sweeps"])
