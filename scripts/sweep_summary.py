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
    if d.get("impl") == "reference":
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

# in-step kernel classes (present when the sweep ran with kernel timing: scripts/sweep_kt.sh)
krows = []
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads([x for x in open(f) if x.startswith("{")][-1])
    except Exception:  # noqa: BLE001
        continue
    k = d.get("kernels") or {}
    if not k:
        continue
    g = lambda n, f_="tflops": (k.get(n) or {}).get(f_) or "-"  # noqa: E731
    tot = sum(v["ms"] for v in k.values()) or 1
    share = lambda n: f"{100 * (k.get(n) or {}).get('ms', 0) / tot:.1f}%"  # noqa: E731
    krows.append(f"| {os.path.basename(f)[:-5]} | {g('gemm_fwd')} | {g('gemm_dgrad')} | {g('gemm_wgrad')} | "
                 f"{g('attn_fwd')} ({share('attn_fwd')}) | {g('attn_bwd')} ({share('attn_bwd')}) | "
                 f"{g('layernorm', 'gbs')} ({share('layernorm')}) |")
if krows:
    print()
    print("| run | GEMM fwd TF/s | dgrad TF/s | wgrad TF/s | attention fwd TF/s (share) | attention bwd TF/s (share) | LayerNorm GB/s (share) |")
    print("|---|---|---|---|---|---|---|")
    print("\n".join(krows))
