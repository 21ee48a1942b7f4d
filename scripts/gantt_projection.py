"""Gantt SVG of the 8-GPU static-order replay of a bench line's measured task costs
(bubble evidence), e.g.  python scripts/gantt_projection.py profiles/r01_bench_1p3b_final.json
profiles/r01_gantt_projected_d8.svg [--no-zero]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import engine as E  # noqa: E402
from paper_2605_29664_b200 import ppsim as P  # noqa: E402
from paper_2605_29664_b200 import projection as PR  # noqa: E402

line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
zero = "--no-zero" not in sys.argv
pj = line["bubble"]["projected_d8_gpus"]
tag = {"F": P.Kind.Forward, "B": P.Kind.Backward, "R": P.Kind.Reduce, "BC": P.Kind.Broadcast, "U": P.Kind.Update}
costs = {}
for k, v in pj["stage_ms"].items():
    kind = "BC" if k.startswith("BC") else k[0]
    costs[(tag[kind], int(k[len(kind):]))] = v * 1e6
if not zero:  # the replicated variant: an Update = the fused optimizer step + the all-reduce
    for s in range(8):
        costs[(P.Kind.Update, s)] = costs[(P.Kind.Broadcast, s)] + costs[(P.Kind.Reduce, s)]
pol = E.RunConfig(depth=8, threshold=32, windows=4, zero=zero).policy()
rep = PR.static_order_replay(pol, 8, costs, pj["gap_us"] * 1e3)
b = float(P.bubble_ratio(rep, 1))
svg = P.gantt_svg(rep, f"AMDP {'ZeRO' if zero else 'all-reduce'} GPT-1.3B, measured task costs replayed on 8 GPUs "
                       f"(windows 1-2, bubble_ratio(tl, 1) = {b:.3f})", 1, 2)
open(sys.argv[2], "w").write(svg)
print(sys.argv[2], b)
