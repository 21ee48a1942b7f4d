"""Schedule path (partition config -> builder -> stage-executor order -> version oracle ->
bubble metric): this repository's C++ library, through its C-ABI, against the reference.

Three layers of evidence:
  * golden fixtures generated from the unmodified reference (tests/golden/sched_golden.json,
    script alongside) — byte-identical timeline_csv (sha256), reports, bubbles;
  * SURVEY Appendix B fingerprints and the reference's own pinned values
    (T/test_engine.cpp:80-94, T/test_builder.cpp:39-110, T/acceptance.cpp:169-181);
  * when oracle/_ref/ppsim_ref is present, a live diff on extra configurations.
"""
import hashlib
import json
import os
import subprocess
from fractions import Fraction

import pytest

from paper_2605_29664_b200 import ppsim as P

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = json.load(open(os.path.join(HERE, "golden", "sched_golden.json")))
REF = os.path.join(ROOT, "oracle", "_ref", "ppsim_ref")


def _costs(s, d):
    v = [Fraction(x) for x in s.split(",")]
    return v * d if len(v) == 1 else v


def _mk(cfg):
    pol, d, dev, fw, bw, up, comm, inj, pipes, thr, M, zero = cfg
    cl = P.ClusterSpec(d, dev, _costs(fw, d), _costs(bw, d), Fraction(up), Fraction(comm))
    pc = P.PolicyConfig(P.policy_from_name(pol), inj, pipes, thr, M, bool(zero))
    return pc, cl


def _run(cfg):
    pc, cl = _mk(cfg)
    return pc, cl, P.simulate(P.build(pc, cl), cl)


@pytest.mark.parametrize("entry", GOLD, ids=lambda e: "-".join(map(str, e["config"])))
def test_timeline_bit_exact_vs_reference_fixture(entry):
    pc, cl, tl = _run(entry["config"])
    csv = P.timeline_csv(tl)
    if "csv" in entry:
        assert csv == entry["csv"]
    assert hashlib.sha256(csv.encode()).hexdigest() == entry["sha256"]
    assert tl.makespan == Fraction(entry["makespan"])
    assert str(P.bubble_ratio(tl, 0)).replace(" ", "") == entry["bubble_w0"] or \
        P.bubble_ratio(tl, 0) == Fraction(entry["bubble_w0"])
    rep = tl.report(pc, warmup=1)
    if entry["bubble_w1"] is not None:
        assert Fraction(rep["bubble_ratio"]) == Fraction(entry["bubble_w1"])
    mm = rep["mismatch"]
    assert mm["max_overall"] == entry["max_mismatch"]
    assert [e for e in mm["entries"] if e[2]] == entry["mismatch_nonzero"]
    wins = [{"window": w["window"], "window_size": w["window_size"],
             "update_count": w["update_count"], "mismatched_minibatches": w["mismatched"]}
            for w in rep["windows"]]
    assert wins == entry["windows"]["windows"]
    assert rep["memory"] == entry["memory"]
    assert rep["causality_issues"] == [] and rep["overlap_issues"] == []


APPENDIX_B = [  # SURVEY.md Appendix B (probe of the reference), AMDP ZeRO uniform T_f = 1
    ((4, 8, 32, 2), 288, 139, "0f521a809f498fe5c21923137afb6ae37200a9b02aa5cacf45fbf7a68e5a8144"),
    ((4, 8, 32, 1), 288, 66, "c4e3ea4aafe4a2cebae4feb79549bdf55804ba7133b48f38f2c59da6c6c31f9a"),
    ((2, 4, 64, 2), 320, 270, "bb610224d2701c4804b2fa11f72eb9139702856aa7c52dd4409e56bba1d52f96"),
    ((2, 4, 64, 1), 320, 130, "959ca851a4c2eb06aa4d0da192504a19aaeeae951d9bf1269f3cdf7f95e9f706"),
    ((4, 16, 256, 2), 2176, 1135, "5c7c590b485bfe80c20be0f12bb4072a41a21c7e91ff4cc2d3579d3ff6b9edaf"),
    ((4, 16, 256, 1), 2176, 514, "5587f5096f10035624796101651b38282b77f138c2e12b0c72eddce09cb545f7"),
    ((8, 32, 512, 2), 8448, 2079, "b4317d4671702a70815051bd3a788f42b7f1caab4bb8a8482818f095c372f1fc"),
    ((8, 32, 512, 1), 8448, 1026, "be24f5d22ea194c4125011b90b1aa1d02670ca332c5066b670c1e4c6d464879d"),
]


@pytest.mark.parametrize("cfg,events,makespan,sha", APPENDIX_B)
def test_appendix_b_fingerprints(cfg, events, makespan, sha):
    d, thr, M, tb = cfg
    cl = P.ClusterSpec.uniform(d, d, 1, tb)
    tl = P.simulate(P.build(P.PolicyConfig(P.Policy.AMDP, 2, d // 2, thr, M, True), cl), cl)
    csv = P.timeline_csv(tl)
    assert csv.count("\n") - 1 == events
    assert tl.makespan == makespan
    assert hashlib.sha256(csv.encode()).hexdigest() == sha


@pytest.mark.parametrize("thr,M,want", [(8, 128, Fraction(197, 876)), (16, 256, Fraction(397, 1760)),
                                        (32, 512, Fraction(137, 524))])
@pytest.mark.parametrize("zero", [False, True])
def test_reference_bubble_pins(thr, M, want, zero):  # T/test_engine.cpp:80-94
    cl = P.ClusterSpec.uniform(8, 8, 1, 2)
    tl = P.simulate(P.build(P.PolicyConfig(P.Policy.AMDP, 2, 4, thr, M, zero), cl), cl)
    assert P.bubble_ratio(tl, 1) == want


def test_mapping_goldens():  # T/test_builder.cpp:39-56, T/acceptance.cpp:169-181
    assert [P.map_stage_to_device(0, i, 8) for i in range(8)] == list(range(8))
    assert [P.map_stage_to_device(1, i, 8) for i in range(8)] == [3, 2, 1, 0, 7, 6, 5, 4]
    assert [P.map_stage_to_device(0, i, 2) for i in range(2)] == [0, 1]
    for d in (2, 4, 8, 16):
        for p in range(d // 2):
            assert sorted(P.map_stage_to_device(p, i, d) for i in range(d)) == list(range(d))
    with pytest.raises(ValueError):
        P.map_stage_to_device(0, 0, 3)
    with pytest.raises(ValueError):
        P.map_stage_to_device(4, 0, 8)


def test_pipelines_and_preload():  # T/test_builder.cpp:89-110
    assert [P.default_num_pipelines(d) for d in (8, 4, 2)] == [4, 2, 1]
    with pytest.raises(ValueError):
        P.default_num_pipelines(5)
    assert P.preload_count(2, 1) == 2
    assert P.preload_count(Fraction(3, 2), 1) == 1
    assert P.preload_count(1, 1) == 1
    assert P.preload_count(Fraction(7, 2), 1) == 3
    assert P.preload_count(Fraction(1, 2), 1) == 0
    with pytest.raises(ValueError):
        P.preload_count(1, 0)


def test_preloaded_sets():  # T/test_builder.cpp:128-171
    for tb, M, want in ((2, 7, {4, 5, 6}), (1, 8, {4, 5})):
        cl = P.ClusterSpec.uniform(4, 4, 1, tb)
        g = P.build(P.PolicyConfig(P.Policy.AMDP, 2, 2, 4, M, True), cl)
        pre = {t.minibatch for t in g.tasks if t.kind == P.Kind.Forward and t.preloaded}
        assert pre == want


def test_named_rejections():  # T/test_builder.cpp:300-323
    cl = P.ClusterSpec.uniform(8, 8, 1, 2)
    with pytest.raises(ValueError, match="invalid configuration: AMDP: num_pipelines must equal depth/2"):
        P.build(P.PolicyConfig(P.Policy.AMDP, 2, 2, 32, 64, True), cl)
    with pytest.raises(ValueError, match="injection_limit is fixed to 2"):
        P.build(P.PolicyConfig(P.Policy.AMDP, 3, 4, 32, 64, True), cl)
    with pytest.raises(ValueError, match="multiple of num_pipelines"):
        P.build(P.PolicyConfig(P.Policy.AMDP, 2, 4, 30, 60, True), cl)
    with pytest.raises(ValueError, match="zero_enabled: only supported for AMDP"):
        P.build(P.PolicyConfig(P.Policy.DAPPLE, 8, 1, 8, 8, True), cl)
    v = P.validate_cluster(P.ClusterSpec(1, 0, [], []))
    assert v[:2] == ["depth: must be >= 2 (got 1)", "devices: must be >= 1 (got 0)"]


def test_dapple_closed_form():  # T/test_engine.cpp:34-43 and T/test_cli.cpp:101-105
    for d, n, tb in ((4, 8, 1), (4, 8, 2), (8, 16, 2)):
        cl = P.ClusterSpec.uniform(d, d, 1, tb)
        tl = P.simulate(P.build(P.PolicyConfig(P.Policy.DAPPLE, n, 1, n, n), cl), cl)
        assert tl.makespan == (n + d - 1) * (1 + tb)
        assert P.bubble_ratio(tl) == Fraction(d - 1, n + d - 1)
    cl = P.ClusterSpec.uniform(4, 4, 1, 2, 0, Fraction(1, 2))
    tl = P.simulate(P.build(P.PolicyConfig(P.Policy.DAPPLE, 8, 1, 8, 8), cl), cl)
    assert tl.makespan == 41 and P.bubble_ratio(tl) == Fraction(17, 41)


def test_cycle_witness_and_deadlock():  # T/test_engine.cpp:192-239
    cl = P.ClusterSpec.uniform(2, 2, 1, 1)
    g = P.TaskGraph(P.Policy.DAPPLE, 2, 2, 1)
    g.tasks = [P.Task(P.Kind.Forward, 0, 0, 0, 0, Fraction(1)), P.Task(P.Kind.Forward, 1, 0, 0, 1, Fraction(1)),
               P.Task(P.Kind.Backward, 1, 0, 0, 1, Fraction(1))]
    g.deps = [(0, 1), (1, 2), (2, 1)]
    with pytest.raises(RuntimeError, match=r"dependency cycle: .*Forward\(stage=1,mb=0,pipe=0\)@dev1"):
        P.simulate(g, cl)
    g.deps = [(0, 1), (1, 2)]
    tl = P.simulate(g, cl)
    assert tl.makespan == 3 and tl.order == [0, 1, 2]


def test_dispatch_order_is_topological_and_versions_structural():
    """The order the GPU executor replays: a linear extension of the DAG; and the parameter
    version each F/B reads is w - preloaded (F) and w (B)."""
    for d, tb in ((4, 1), (8, 1), (8, 2)):
        thr = 4 * d
        cl = P.ClusterSpec.uniform(d, d, 1, tb)
        g = P.build(P.PolicyConfig(P.Policy.AMDP, 2, d // 2, thr, 4 * thr, True), cl)
        tl = P.simulate(g, cl)
        pos = {t: i for i, t in enumerate(tl.order)}
        assert all(pos[a] < pos[b] for a, b in g.deps)
        rows = P.version_trace_csv(tl).strip().split("\n")[1:]
        for r in rows:
            dev, kind, stage, mb, pipe, w, pre, ver = r.split(",")
            want = int(w) - int(pre) if kind == "Forward" else int(w)
            assert int(ver) == want, r


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", [
    ("AMDP", 8, 8, "1", "9/5", "0", "0", 2, 4, 16, 96, 1),
    ("AMDP", 4, 4, "2", "3", "1/3", "1/7", 2, 2, 4, 40, 0),
    ("AMDP", 10, 10, "1", "2", "0", "0", 2, 5, 10, 50, 1),
    ("Chimera", 6, 6, "1", "2", "0", "1/2", 6, 2, 6, 18, 0),
    ("Interleaved1F1B", 4, 2, "1", "2", "0", "0", 4, 1, 4, 12, 0),
])
def test_live_reference_diff(cfg):
    args = [REF] + [str(x) for x in cfg] + ["csv"]
    ref = subprocess.run(args, check=True, capture_output=True, text=True).stdout
    assert P.timeline_csv(_run(cfg)[2]) == ref
