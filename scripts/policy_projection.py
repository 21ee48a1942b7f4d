"""Paper Table-2-style comparison on B200 stage costs: projects AMDP, DAPPLE, GPipe, Chimera and
PipeDreamAsync at D GPUs from per-stage Forward / Backward / optimizer costs measured by bench.py
on one B200 (the `stage_ms` of its `projected_dD_gpus` entry).  CPU only.

    python scripts/policy_projection.py profiles/r01_bench_1p3b_final.json [windows]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import ppsim as P
from paper_2605_29664_b200 import projection as PR

line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
windows = int(sys.argv[2]) if len(sys.argv) > 2 else 6
key = [k for k in line["bubble"] if k.startswith("projected")][0]
proj = line["bubble"][key]
tags = {v: k for k, v in PR.KIND_TAG.items()}
costs = {}
for k, v in proj["stage_ms"].items():
    tag = k.rstrip("0123456789")
    if tag in tags:
        costs[(tags[tag], int(k[len(tag):]))] = v * 1e6
depth = max(s for (_, s) in costs) + 1
opt = line.get("kernels", {}).get("optimizer")  # older lines: optimizer cost from the kernel table
if opt and opt.get("launches"):
    for s_ in range(depth):
        costs.setdefault((P.Kind.Broadcast, s_), opt["ms"] / opt["launches"] * 1e6)
thr = line["config"]["global_batch"] // 4  # 4 sequences per minibatch
tpm = line["config"]["tokens_per_step"] // thr
res = PR.compare_policies(costs, depth, thr, windows, tpm, proj["gap_us"] * 1e3)
print(json.dumps({"source": sys.argv[1], "depth": depth, "threshold": thr, "windows": windows,
                  "gap_us": proj["gap_us"], "policies": res}, indent=1))
