"""Markdown table of a bench.py sweep directory (scripts/sweep.sh)."""
import glob
import json
import os
import sys

rows = []
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads([x for x in open(f) if x.startswith("{")][-1])
    except Exception:  # noqa: BLE001
        continue
    c = d["config"]
    pr = next((v for k, v in d["bubble"].items() if k.startswith("projected_")), None) or {}
    alt = pr.get("allreduce_update_variant") or {}
    f3 = lambda x: "-" if x is None else f"{x:.4f}"  # noqa: E731
    rows.append(f"| {os.path.basename(f)[:-5]} | {c['model']} | {c['parallelism']} | {d['value']:.0f} | {d['e2e']['value']:.0f} | "
                f"{d['model_flops_utilization']:.3f} / {d['model_flops_vs_measured_sustained_peak']:.3f} | {f3(pr.get('bubble'))} | "
                f"{f3(alt.get('bubble'))} | {pr.get('tokens_per_s') or 0:.0f} | {d['clocks']['sm_mhz']} | {d['memory_gb']['total']} |")
print("| run | model | parallelism | tokens/s (1 GPU) | e2e | MFU (spec / sustained) | projected bubble (ZeRO) | "
      "projected bubble (all-reduce updates) | projected tokens/s at D GPUs | SM MHz | memory GB |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
