"""Projection of a measured 1-GPU run onto d GPUs (one logical device each).

The executor replays the schedule's declared dispatch order (`simulate` on the declared cost
model).  On d GPUs every device would run its own tasks in that same
order, so the multi-GPU timeline follows from a static-order replay: walk the declared
global order and re-time each task with its MEASURED cost,

    start = max(device free, max over predecessors (finish + gap(dev_pred, dev)))

where the gap is the inter-stage activation transfer (bytes / link bandwidth).  The result
feeds the reference's own `bubble_ratio` (engine.hpp:166-202).  This is a projection from
measured per-stage costs, not a multi-GPU measurement (this pool grants one GPU).
"""
from __future__ import annotations

import statistics
from fractions import Fraction
from typing import Dict, Tuple

from . import ppsim as P

# per-stage cost keys in bench.py's JSON: F3 = Forward of stage 3, BC3 = Broadcast (optimizer) ...
KIND_TAG = {P.Kind.Forward: "F", P.Kind.Backward: "B", P.Kind.Reduce: "R", P.Kind.Broadcast: "BC",
            P.Kind.Update: "U"}


def measured_costs(tl: P.Timeline, min_window: int = 1, lane_events=None) -> Dict[Tuple[P.Kind, int], float]:
    """Mean measured duration (ns) per (kind, stage) over windows >= min_window.  Update tasks
    take the max: folded on one GPU only the first replica's Update of a window runs the
    optimizer (the others switch weight buffers), while on one GPU per device every replica
    steps its own optimizer state.  `lane_events` (Engine.lane_events()): the Reduce /
    Broadcast intervals on the executor's collective / update streams, which replace the
    compute-stream markers of those tasks."""
    acc: Dict[Tuple[P.Kind, int], list] = {}
    lane_kinds = {ev.kind for ev in lane_events} if lane_events else set()
    for ev in tl.flat():
        if ev.window >= min_window and ev.kind not in lane_kinds:
            acc.setdefault((ev.kind, ev.stage), []).append(float(ev.duration))
    for ev in lane_events or []:
        if ev.window >= min_window:
            acc.setdefault((ev.kind, ev.stage), []).append(float(ev.duration))
    return {k: (max(v) if k[0] == P.Kind.Update else statistics.mean(v)) for k, v in acc.items()}


def static_order_replay(policy: P.PolicyConfig, depth: int, costs_ns: Dict[Tuple[P.Kind, int], float],
                        gap_ns: float, declared_fwd=1, declared_bwd=1, devices: int = 0,
                        update_lane: bool = False, lane_out: dict = None, segments=None) -> P.Timeline:
    """Re-times the declared dispatch order of `policy` (depth stages on `devices`, default
    depth) with measured costs.  Update tasks (replicated-weight policies) cost what the
    stage's measured Broadcast (fused optimizer step) cost.

    update_lane: the executor's ZeRO window machinery — Reduce on a collective stream and
    Broadcast (optimizer + weight broadcast) on an update stream.  Such a task starts once
    its graph predecessors have finished AND the device's compute stream has reached its
    position in the order (the executor hands the compute stream's progress to it), but it
    does not hold the compute stream: only its graph successors (BC(w-1,i) -> F / preloaded
    B, builder.hpp:289-304) wait for it.  In the returned timeline these tasks are
    zero-length at their finish, so `bubble_ratio` measures compute-stream idle time; their
    real intervals are appended to `lane_out["events"]` if given.

    segments (per stage, with update_lane): the Broadcast steps the optimizer segment by
    segment (embeddings, each layer, head) in the forward's reading order and a gated Forward
    waits per segment: it may start once the first segment is stepped and cannot finish
    earlier than one segment's share of its own cost after the last one (the optimizer part
    taken as 90% of the Broadcast, the rest being the backward's transposed copies)."""
    devices = devices or depth
    declared = P.ClusterSpec.uniform(depth, devices, declared_fwd, declared_bwd)
    g = P.build(policy, declared)
    tl = P.simulate(g, declared)
    costs_ns = dict(costs_ns)
    for s in range(depth):
        if (P.Kind.Update, s) not in costs_ns and (P.Kind.Broadcast, s) in costs_ns:
            costs_ns[(P.Kind.Update, s)] = costs_ns[(P.Kind.Broadcast, s)]
    preds = [[] for _ in g.tasks]
    for a, b in g.deps:
        preds[b].append(a)
    free = [0] * devices
    ufree = [0] * devices
    finish = [0] * len(g.tasks)
    bc_start = [0] * len(g.tasks)
    gap = int(round(gap_ns))
    events = []
    lane_kinds = (P.Kind.Reduce, P.Kind.Broadcast) if update_lane else ()
    for t in tl.order:
        task = g.tasks[t]
        dur = int(round(costs_ns.get((task.kind, task.stage), 0.0)))
        on_lane = task.kind in lane_kinds
        start = max(free[task.device], ufree[task.device]) if on_lane else free[task.device]
        min_finish = 0
        for p in preds[t]:
            ready = finish[p] + (gap if g.tasks[p].device != task.device else 0)
            if segments and task.kind == P.Kind.Forward and g.tasks[p].kind == P.Kind.Broadcast:
                nseg = segments[task.stage]
                opt = 0.9 * (finish[p] - bc_start[p])
                ready = bc_start[p] + opt / nseg
                min_finish = max(min_finish, bc_start[p] + opt + dur / nseg)
            start = max(start, ready)
        finish[t] = max(start + dur, min_finish)
        dur = finish[t] - start
        bc_start[t] = start
        if on_lane:
            ufree[task.device] = finish[t]
            if lane_out is not None:
                lane_out.setdefault("events", []).append((task.kind, task.stage, task.device, start, dur))
            events.append(P.TaskEvent(task.kind, task.stage, task.minibatch, task.pipeline, task.device,
                                      Fraction(finish[t]), Fraction(0), task.preloaded, task.window))
            continue
        free[task.device] = finish[t]
        events.append(P.TaskEvent(task.kind, task.stage, task.minibatch, task.pipeline, task.device,
                                  Fraction(start), Fraction(dur), task.preloaded, task.window))
    return P.Timeline.from_events(events, policy.policy, depth, devices, policy.accumulation_threshold)


def collective_costs(stage_numel, replicas: int, link_gbs: float = 770.0,
                     zero: bool = True) -> Dict[Tuple[P.Kind, int], float]:
    """Window-boundary communication a 1-GPU run does not perform.  ZeRO (the executor's
    peer-memory data plane): the Reduce is a reduce-scatter of the fp32 window gradient
    (4 B/param) and the Broadcast an all-gather of the bf16 weights (2 B/param; the LayerNorm
    parameters' fp32 copy is negligible) over the stage's `replicas` devices, each device
    pulling (replicas-1)/replicas of those bytes (analysis.hpp:341-346 reduce_broadcast_cost)
    at the measured peer bandwidth; without ZeRO, the all-reduce of the fp32 window gradient
    (reduce-scatter + all-gather volume) in every Update."""
    f = (replicas - 1) / replicas if replicas > 1 else 0.0
    out = {}
    for s, n in enumerate(stage_numel):
        t = f * 4.0 * n / (link_gbs * 1e9) * 1e9
        if zero:
            out[(P.Kind.Reduce, s)] = t
            out[(P.Kind.Broadcast, s)] = t / 2
        else:
            out[(P.Kind.Update, s)] = 2 * t
    return out


def replicas_of(policy: P.PolicyConfig) -> int:
    """Weight replicas per stage (builder.hpp:154-156): AMDP d/2 pipelines, Chimera 2, else 1."""
    if policy.policy == P.Policy.AMDP:
        return policy.num_pipelines
    return 2 if policy.policy == P.Policy.Chimera else 1


def project(tl_measured: P.Timeline, depth: int, threshold: int, windows: int, tokens_per_minibatch: int,
            gap_ns: float, stage_numel=None, policy: P.PolicyConfig = None, lane_events=None,
            segments=None) -> dict:
    """Projected d-GPU bubble and throughput of a measured run's schedule (default AMDP).  With
    `stage_numel`, the Reduce / Broadcast tasks also carry the NVLink collective time
    (collective_costs) on top of what was measured on one GPU (the fused optimizer)."""
    costs = measured_costs(tl_measured, lane_events=lane_events)
    pol = policy or P.PolicyConfig(policy=P.Policy.AMDP, injection_limit=2, num_pipelines=depth // 2,
                                   accumulation_threshold=threshold, num_minibatches=windows * threshold,
                                   zero_enabled=True)
    bubble_nc = None
    devices = depth // 2 if pol.policy == P.Policy.Interleaved1F1B else depth
    for s in range(depth):  # an Update steps the optimizer: a ZeRO run measured that as Broadcast
        if (P.Kind.Update, s) not in costs and (P.Kind.Broadcast, s) in costs:
            costs[(P.Kind.Update, s)] = costs[(P.Kind.Broadcast, s)]
    lane = bool(pol.zero_enabled)  # the executor's update / collective streams (ZeRO)
    if lane and replicas_of(pol) > 1:
        # ZeRO within the replica group on d GPUs: each of the P replicas steps the optimizer on
        # 1/P of the stage (the measured 1-GPU Broadcast stepped all of it); the transposed
        # weight refresh (4 of the Broadcast's ~38 bytes per parameter, ~10%) stays whole
        P_ = replicas_of(pol)
        for s_ in range(depth):
            if (P.Kind.Broadcast, s_) in costs:
                costs[(P.Kind.Broadcast, s_)] *= 0.9 / P_ + 0.1
    if stage_numel is not None and replicas_of(pol) > 1:
        rep0 = static_order_replay(pol, depth, costs, gap_ns, devices=devices, update_lane=lane,
                                   segments=segments if lane else None)
        bubble_nc = float(P.bubble_ratio(rep0, 1 if windows > 2 else 0))
        for k, v in collective_costs(stage_numel, replicas_of(pol), zero=pol.zero_enabled).items():
            costs[k] = costs.get(k, 0.0) + v
    lane_out = {}
    rep = static_order_replay(pol, depth, costs, gap_ns, devices=devices, update_lane=lane, lane_out=lane_out,
                              segments=segments if lane else None)
    bubble = P.bubble_ratio(rep, 1 if windows > 2 else 0)
    # the same costs with the window machinery serialised on the compute stream (round-1 executor)
    serial = static_order_replay(pol, depth, costs, gap_ns, devices=devices) if lane else rep
    bubble_serial = float(P.bubble_ratio(serial, 1 if windows > 2 else 0))
    # steady-state window period: first F of window w to first F of window w+1, averaged
    firsts = {}
    for ev in rep.flat():
        if ev.kind == P.Kind.Forward:
            firsts[ev.window] = min(firsts.get(ev.window, ev.start), ev.start)
    ws = sorted(firsts)
    period = float(firsts[ws[-1]] - firsts[ws[1]]) / (len(ws) - 2) if len(ws) > 2 else None
    return {"gpus": devices, "bubble": float(bubble), "bubble_without_collectives": bubble_nc,
            "bubble_window_machinery_serialised": bubble_serial,
            "update_lane": "Reduce / Broadcast on the collective / update streams, off the compute stream"
                           if lane else "Update tasks on the compute stream",
            "tokens_per_s": (threshold * tokens_per_minibatch / (period * 1e-9)) if period else None,
            "gap_us": gap_ns / 1e3,
            "stage_ms": {f"{KIND_TAG[k[0]]}{k[1]}": round(v / 1e6, 3) for k, v in sorted(costs.items())},
            "method": "static-order replay of the declared dispatch order on one GPU per "
                      "logical device, task costs = measured 1-GPU means (windows >= 1) plus the "
                      "window Reduce (fp32) / Broadcast (bf16) collectives (or the replicated Update's "
                      "all-reduce) at 770 GB/s ((P-1)/P of the stage's bytes per phase); ZeRO Reduce / "
                      "Broadcast on the update lane (start when the compute stream reaches them, only "
                      "their graph successors wait); inter-device gap = activation bytes / 770 GB/s peer "
                      "copy; bubble = reference bubble_ratio(tl, 1) of the compute streams.  A projection, "
                      "not a multi-GPU measurement."}


# Schedules of the paper's comparison (reference builder.hpp policies) on the same D stages /
# D devices, thr minibatches per accumulation window.  Interleaved 1F1B needs
# 2D stages (another partition) and is left out.
COMPARE = {
    "AMDP": lambda d, thr, m: P.PolicyConfig(P.Policy.AMDP, 2, d // 2, thr, m, True),
    # synchronous schedules inject the whole window (validate.hpp: threshold == injection limit)
    "DAPPLE": lambda d, thr, m: P.PolicyConfig(P.Policy.DAPPLE, thr, 1, thr, m, False),
    "GPipe": lambda d, thr, m: P.PolicyConfig(P.Policy.GPipe, thr, 1, thr, m, False),
    "Chimera": lambda d, thr, m: P.PolicyConfig(P.Policy.Chimera, thr, 2, thr, m, False),
    "PipeDreamAsync": lambda d, thr, m: P.PolicyConfig(P.Policy.PipeDreamAsync, d, 1, thr, m, False),
}


def compare_policies(costs_ns: Dict[Tuple[P.Kind, int], float], depth: int, threshold: int, windows: int,
                     tokens_per_minibatch: int, gap_ns: float) -> dict:
    """Projected bubble / tokens/s / makespan of each policy from the same measured stage costs."""
    out = {}
    for name, mk in COMPARE.items():
        pol = mk(depth, threshold, windows * threshold)
        try:
            rep = static_order_replay(pol, depth, costs_ns, gap_ns)
        except Exception as e:  # a policy whose rules reject this shape
            out[name] = {"error": str(e)[:160]}
            continue
        ev = rep.flat()
        span = float(max(e.finish() for e in ev))
        out[name] = {"bubble_w1": float(P.bubble_ratio(rep, 1 if windows > 2 else 0)),
                     "tokens_per_s": windows * threshold * tokens_per_minibatch / (span * 1e-9),
                     "makespan_ms": span / 1e6}
    return out
