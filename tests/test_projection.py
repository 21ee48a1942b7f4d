"""Static-order replay projection (paper_2605_29664_b200/projection.py), CPU only.

With task costs equal to the declared cost model and no gap, re-timing the declared
dispatch order must reproduce `simulate` exactly (the executor's order is a list schedule
of those costs); with slower backward or an inter-device gap the replay can only get
longer, and its events must satisfy the reference's causality / non-overlap validators."""
from fractions import Fraction

import pytest

from paper_2605_29664_b200 import ppsim as P
from paper_2605_29664_b200 import projection as PR


def _pol(d, thr, windows):
    return P.PolicyConfig(P.Policy.AMDP, 2, d // 2, thr, windows * thr, True)


@pytest.mark.parametrize("d,thr,windows", [(4, 8, 3), (8, 32, 3), (2, 4, 4)])
def test_replay_with_declared_costs_is_simulate(d, thr, windows):
    pol = _pol(d, thr, windows)
    costs = {(k, s): 1000.0 for k in (P.Kind.Forward, P.Kind.Backward) for s in range(d)}
    rep = PR.static_order_replay(pol, d, costs, 0.0)
    decl = P.ClusterSpec.uniform(d, d, 1, 1)
    sim = P.simulate(P.build(pol, decl), decl)
    a = sorted((e.device, e.kind, e.stage, e.minibatch, e.pipeline, e.start, e.duration) for e in rep.flat())
    b = sorted((e.device, e.kind, e.stage, e.minibatch, e.pipeline, e.start * 1000, e.duration * 1000)
               for e in sim.flat())
    assert a == b
    assert P.bubble_ratio(rep, 1) == P.bubble_ratio(sim, 1)


def test_replay_slower_backward_and_gap_is_causal():
    d, thr, windows = 8, 32, 3
    pol = _pol(d, thr, windows)
    costs = {}
    for s in range(d):
        costs[(P.Kind.Forward, s)] = 1000.0
        costs[(P.Kind.Backward, s)] = 2100.0
    base = PR.static_order_replay(pol, d, {k: 1000.0 for k in costs}, 0.0)
    rep = PR.static_order_replay(pol, d, costs, 50.0)
    cl = P.ClusterSpec(d, d, [Fraction(1000)] * d, [Fraction(2100)] * d, Fraction(0), Fraction(50))
    assert P.validate_causality(rep, cl) == []
    assert P.validate_non_overlap(rep) == []
    assert max(e.finish() for e in rep.flat()) > max(e.finish() for e in base.flat())
    assert 0 <= P.bubble_ratio(rep, 1) < 1


def test_compare_policies_all_schedules_run_and_amdp_matches_project():
    d, thr, windows = 8, 32, 3
    costs = {}
    for s in range(d):
        costs[(P.Kind.Forward, s)] = 1000.0 + 100 * (s < 2)
        costs[(P.Kind.Backward, s)] = 2200.0 + 200 * (s < 2)
        costs[(P.Kind.Broadcast, s)] = 300.0
    res = PR.compare_policies(costs, d, thr, windows, 8192, 40.0)
    assert set(res) == {"AMDP", "DAPPLE", "GPipe", "Chimera", "PipeDreamAsync"}
    for name, r in res.items():
        assert "error" not in r, (name, r)
        assert 0 <= r["bubble_w1"] < 1 and r["tokens_per_s"] > 0
    rep = PR.static_order_replay(_pol(d, thr, windows), d, costs, 40.0)
    assert abs(float(P.bubble_ratio(rep, 1)) - res["AMDP"]["bubble_w1"]) < 1e-12


def test_collective_costs_follow_reduce_broadcast_cost():
    # (P-1)/P of the stage's fp32 bytes per phase at the link bandwidth (analysis.hpp:341-346)
    c = PR.collective_costs([1_000_000, 2_000_000], 4, link_gbs=1000.0)
    assert abs(c[(P.Kind.Reduce, 0)] - 0.75 * 4e6 / 1e12 * 1e9) < 1e-6
    assert c[(P.Kind.Broadcast, 1)] == 2 * c[(P.Kind.Broadcast, 0)]
    assert PR.collective_costs([5], 1) == {(P.Kind.Reduce, 0): 0.0, (P.Kind.Broadcast, 0): 0.0}


def test_gantt_svg_renders_every_task():
    """ppsim.gantt_svg (the gantt.hpp view): valid SVG, one bar per task of non-zero duration,
    deterministic."""
    import xml.etree.ElementTree as ET
    cl = P.ClusterSpec.uniform(4, 4, 1, 2)
    tl = P.simulate(P.build(P.PolicyConfig(P.Policy.AMDP, 2, 2, 8, 32, True), cl), cl)
    svg = P.gantt_svg(tl)
    assert svg == P.gantt_svg(tl)
    root = ET.fromstring(svg)
    bars = [r for r in root.iter("{http://www.w3.org/2000/svg}rect") if r.find("{http://www.w3.org/2000/svg}title") is not None]
    assert len(bars) == sum(1 for e in tl.flat() if e.duration > 0)


def test_update_lane_takes_window_machinery_off_the_compute_stream():
    """ZeRO Reduce / Broadcast on the update lane (the executor's collective / update streams):
    they start only after their graph predecessors and the device's compute up to their order
    position, every successor (BC(w-1,i) -> F / preloaded B) still waits for them, and the
    compute-stream bubble is no larger than with the machinery serialised on the compute stream."""
    d, thr, windows = 8, 32, 4
    pol = _pol(d, thr, windows)
    costs = {}
    for s in range(d):
        costs[(P.Kind.Forward, s)] = 1000.0
        costs[(P.Kind.Backward, s)] = 2000.0
        costs[(P.Kind.Reduce, s)] = 400.0
        costs[(P.Kind.Broadcast, s)] = 900.0
    lane = {}
    rep = PR.static_order_replay(pol, d, costs, 30.0, update_lane=True, lane_out=lane)
    ser = PR.static_order_replay(pol, d, costs, 30.0)
    assert P.bubble_ratio(rep, 1) <= P.bubble_ratio(ser, 1)
    assert max(e.finish() for e in rep.flat()) <= max(e.finish() for e in ser.flat())
    g = P.build(pol, P.ClusterSpec.uniform(d, d, 1, 1))
    fin = {}
    for e in rep.flat():
        fin[(e.kind, e.stage, e.minibatch, e.pipeline)] = e.finish()
    # lane tasks appear as zero-length events at their finish; their successors start after it
    for a, b in g.deps:
        ta, tb = g.tasks[a], g.tasks[b]
        if ta.kind == P.Kind.Broadcast:
            fa = fin[(ta.kind, ta.stage, ta.minibatch, ta.pipeline)]
            sb = next(e.start for e in rep.flat() if (e.kind, e.stage, e.minibatch, e.pipeline) ==
                      (tb.kind, tb.stage, tb.minibatch, tb.pipeline))
            assert sb >= fa
    assert len(lane["events"]) == 2 * d * windows
    assert all(dur in (400, 900) for (_, _, _, _, dur) in lane["events"])
