"""Gantt SVG of the 8-GPU static-order replay of a bench line's projected task costs (bubble
evidence).  The ZeRO window machinery is drawn on its own lane under each device ("upd d"):
Reduce (reduce-scatter) and Broadcast (sharded optimizer step + all-gather) run on the update /
collective streams beside the compute stream; only the tasks they gate wait for them.

    python scripts/gantt_projection.py profiles/r02/bench_1p3b_zero_sharded.json \
        profiles/r02_gantt_projected_d8_zero.svg
"""
import json
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import engine as E  # noqa: E402
from paper_2605_29664_b200 import ppsim as P  # noqa: E402
from paper_2605_29664_b200 import projection as PR  # noqa: E402

line = json.loads([x for x in open(sys.argv[1]) if x.startswith("{")][-1])
pj = line["bubble"]["projected_d8_gpus"]
tag = {"F": P.Kind.Forward, "B": P.Kind.Backward, "R": P.Kind.Reduce, "BC": P.Kind.Broadcast, "U": P.Kind.Update}
costs = {}
for k, v in pj["stage_ms"].items():  # already the projection's costs (shards, collectives)
    kind = "BC" if k.startswith("BC") else k[0]
    costs[(tag[kind], int(k[len(kind):]))] = v * 1e6
part = [4, 3, 3, 3, 3, 3, 3, 2]
segs = [part[i] + (i == 0) + (i == 7) for i in range(8)]
pol = E.RunConfig(depth=8, threshold=32, windows=4).policy()
lane = {}
rep = PR.static_order_replay(pol, 8, costs, pj["gap_us"] * 1e3, update_lane=True, lane_out=lane, segments=segs)
b = float(P.bubble_ratio(rep, 1))
# compute lanes 0-7 (the replay), update lanes 8-15 (the window machinery's intervals)
evs = [e for e in rep.flat() if e.kind in (P.Kind.Forward, P.Kind.Backward)]
for (kind, stage, dev, start, dur) in lane["events"]:
    w = next(e.window for e in rep.flat() if e.kind == kind and e.stage == stage and e.device == dev
             and e.start >= start)
    evs.append(P.TaskEvent(kind, stage, 0, 0, 8 + dev, Fraction(start), Fraction(dur), False, w))
tl = P.Timeline.from_events(evs, pol.policy, 8, 16, 32)
svg = P.gantt_svg(tl, f"AMDP ZeRO GPT-1.3B, projected task costs replayed on 8 GPUs (windows 1-2; lanes 8-15 = "
                      f"update/collective streams of devices 0-7; compute bubble_ratio(tl, 1) = {b:.3f})", 1, 2)
open(sys.argv[2], "w").write(svg)
print(sys.argv[2], b)
