"""AMDP training throughput on B200: GPT-style 1.3B, D=8 logical stages, 4 multi-directional
pipelines, 32 minibatches (4 x 2048 tokens) per optimizer step (BASELINE.json configs[3]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

A "step" is one accumulation window of the AMDP schedule: 32 minibatches x 8192 tokens =
262,144 tokens, every stage forward + backward + the window's Reduce/Broadcast (fused
optimizer step).  The 8 logical devices (AMDP needs devices == depth) are folded onto the N
GPUs (8/N per GPU); N=1 runs all stages time-multiplexed on one B200.

Timed regions (device-timed with CUDA events on the engine's compute stream; barrier +
synchronize on both sides; max over ranks):
  value : K windows run from an empty pipeline with tokens already resident in HBM;
  e2e   : the same K windows through the public API with pinned-host token arrays —
          every window's host->device token copy and the device->host loss read are inside
          the (wall-clock) timed region;
  kernel classes (roofline) : a third run with per-launch CUDA events.
The working set (activations, GBs) exceeds the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPEC_BF16_TFLOPS = 2250.0  # dense bf16 tensor-core peak per B200 (spec sheet; 4.5 PF is 2:4 sparse)
PEAK_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return dict(PEAK_FALLBACK), "fallback"


# Model shapes (layers, hidden, heads, ffn, vocab, seq, causal) — the same as
# paper_2605_29664_b200.engine.ModelConfig's factories, restated here so that the reference
# arm (--impl reference) never imports the product package or loads libamdp.so.
MODELS = {"1p3b": (24, 2048, 16, 8192, 50304, 2048, True), "350m": (24, 1024, 16, 4096, 50304, 1024, True),
          "2p7b": (32, 2560, 32, 10240, 50304, 2048, True), "bert": (24, 1024, 16, 4096, 30528, 512, False),
          "tiny": (4, 128, 4, 512, 1024, 64, True)}


def flops_per_token(name):
    """Training FLOPs per token, 6 L (4h^2 + 2 h ffn) + 12 L s h + 6 h V."""
    L, h, _, f, V, s, _ = MODELS[name]
    return 6 * L * (4 * h * h + 2 * h * f) + 12 * L * s * h + 6 * h * V


def model_cfg(name):
    from paper_2605_29664_b200 import engine as E
    L, h, H, f, V, s, causal = MODELS[name]
    return E.ModelConfig(L, h, H, f, V, s, causal=causal)


class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 4:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), float(parts[2]), int(parts[3], 16)))
                except ValueError:
                    pass

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        load = [r for r in rows if r[2] > 200] or rows
        bits = 0
        for r in load:
            bits |= r[3]
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows), "power_w_median": statistics.median(r[2] for r in load),
                "samples": len(load),
                "reasons": [n for b, n in names.items() if bits & b and n != "gpu_idle"]}


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import gpt_oracle as O
    return O


class LayerSample:
    """The CPU restatement (oracle/gpt_oracle.py, numpy fp32, all host threads through BLAS) on a
    bounded sample of the workload: forward + backward of ONE transformer layer of the model on
    ONE sequence.  Model-equivalent tokens/s = the sample's FLOP rate / the model's FLOPs per
    token (an extrapolation: kind "port-extrapolated")."""

    def __init__(self, name):
        import numpy as np
        O = _oracle()
        L, h, H, f, V, s, causal = MODELS[name]
        self.name, self.layers, self.seq = name, L, s
        om = O.Model(L, h, H, f, V, s, 1, causal, 1234)
        self.st = O.StageMath(om, 1, 3, 0, 1, emulate_bf16=False)
        self.st.rb = lambda a: np.asarray(a, np.float32)
        self.W = {k: v.astype(np.float32) for k, v in O.init_stage(om, O.stage_param_specs(om, 1, 3, 0, 1)).items()}
        rng = np.random.default_rng(0)
        self.x = rng.standard_normal((s, h)).astype(np.float32)
        self.g = rng.standard_normal((s, h)).astype(np.float32) * 1e-3
        self.grads = {k: np.zeros_like(v) for k, v in self.W.items()}
        self.flops = 3 * (2 * s * (4 * h * h + 2 * h * f) + 2 * s * s * h)  # fwd+bwd, 1 layer, 1 seq

    def step(self):
        _, cache, _ = self.st.forward(self.W, self.x, None, None)
        self.st.backward(self.W, cache, self.g, None, self.grads)

    def describe(self, reps, secs):
        return (f"numpy fp32 forward+backward of 1 of {self.layers} layers on 1 sequence of {self.seq} tokens "
                f"x {reps} samples ({secs:.1f} s); model tokens/s = sample FLOP/s / model FLOPs per token "
                f"({flops_per_token(self.name):.3e})")


def cpu_port_baseline(name, seconds=12.0):
    """Bounded 1-layer sample (LayerSample), repeated for ~`seconds`."""
    smp = LayerSample(name)
    reps, t0 = 0, time.perf_counter()
    while True:
        smp.step()
        reps += 1
        if time.perf_counter() - t0 > seconds or reps >= 50:
            break
    dt = time.perf_counter() - t0
    rate = smp.flops * reps / dt
    return {"value": rate / flops_per_token(name), "unit": "tokens/s", "cores": os.cpu_count(),
            "kind": "port-extrapolated", "sample": smp.describe(reps, dt), "cpu_gflops": rate / 1e9}


def cpu_schedule_replay():
    """A real timed run of the reference path on the CPU: the oracle replays the UNMODIFIED
    reference's AMDP timeline (tests/golden fixture from oracle/_ref/ppsim_ref: tiny GPT,
    D=4, 2 pipelines, 8 minibatches per window) with the reference's version semantics, every
    stage forward/backward and the window optimizer steps, fp64 (numpy, all host threads)."""
    O = _oracle()
    cfg = ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 1]
    with open(os.path.join(ROOT, "tests", "golden", "sched_golden.json")) as f:
        trace = next(e["csv"] for e in json.load(f) if e["config"] == cfg)
    L, h, H, ff, V, s, causal = MODELS["tiny"]
    om = O.Model(L, h, H, ff, V, s, 4, causal, 1234)
    M = 8 * 4
    inputs, labels = O.synthetic_tokens(s, 4, V, 1234, 0, M)
    t0 = time.perf_counter()
    O.replay(trace, om, [1, 1, 1, 1], O.Opt("adamw", 1e-3, 0.9, 0.95, 1e-8, 0.0), 8, inputs, labels)
    dt = time.perf_counter() - t0
    return {"value": M * om.T / dt, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "seconds": dt, "sample": f"oracle replay of the reference AMDP timeline, tiny GPT (L4 h128 seq64), "
                                     f"D=4, 4 windows x 8 minibatches x {om.T} tokens, fp64, all {M} minibatches"}


def schedule_baseline():
    """The reference's own CPU path (ppsim build + simulate + mismatch_report, single-threaded
    as designed) on this workload's schedule, from oracle/_ref when it was built."""
    ref = os.path.join(ROOT, "oracle", "_ref", "ppsim_ref")
    if not os.path.exists(ref):
        return None
    out = subprocess.run([ref, "AMDP", "8", "8", "1", "1", "0", "0", "2", "4", "32", "512", "1", "bench", "20"],
                         capture_output=True, text=True)
    try:
        r = json.loads(out.stdout)
        return {"ms_per_schedule": 1e3 * r["seconds"] / r["reps"], "minibatches": 512, "threads": 1}
    except Exception:
        return None


def lib_numel(eng, stage):
    from paper_2605_29664_b200 import engine as E
    return int(E.lib.amdp_engine_stage_numel(eng._h, stage))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="1p3b")
    ap.add_argument("--threshold", type=int, default=32)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--schedule", default="AMDP",
                    choices=["AMDP", "DAPPLE", "GPipe", "Chimera", "Interleaved1F1B", "PipeDreamAsync"],
                    help="AMDP (headline) or another reference schedule on the same executor")
    ap.add_argument("--no-zero", action="store_true",
                    help="AMDP with replicated per-pipeline updates instead of ZeRO reduce/broadcast")
    ap.add_argument("--no-kernel-timing", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="issue every run eagerly (no CUDA graphs)")
    ap.add_argument("--comm", default="ipc", choices=["ipc", "nccl"],
                    help="N>1 data plane: this library's CUDA-IPC peer-memory backend or NCCL")
    ap.add_argument("--recompute", action="store_true",
                    help="backward rebuilds f = gelu(u) and o = attention(qkv) (fits GPT-2.7B D=8 on one GPU)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    L, h, H, ffn, V, seq, causal = MODELS[args.model]
    tokens_per_mb = 4 * seq
    tok_step = args.threshold * tokens_per_mb
    npipe = {"AMDP": args.depth // 2, "Chimera": 2}.get(args.schedule, 1)
    zero = args.schedule == "AMDP" and not args.no_zero
    cfg = {"workload": f"GPT-style {args.model} {args.schedule} D={args.depth} ({npipe} pipelines), "
                       f"seq {seq}, 4 seqs/minibatch, {args.threshold} minibatches/step",
           "model": ("bert-large" if args.model == "bert" else f"gpt-{args.model}"), "layers": L, "hidden": h,
           "global_batch": args.threshold * 4, "seq_len": seq,
           "tokens_per_step": tok_step, "parallelism": f"{args.schedule.lower()}{'' if zero or args.schedule != 'AMDP' else '-replicated'}-d{args.depth}-p{npipe} folded on {args.gpus} GPU",
           "declared_costs": "uniform fwd=1 bwd=1 (preload 1)", "recompute_f_and_o": bool(args.recompute), "l2": "working set >> L2 (no flush)"}
    metric = "tokens/s AMDP GPT-style training" if args.schedule == "AMDP" else f"tokens/s {args.schedule} GPT-style training"

    if args.impl == "reference":
        # The reference (ppsim) is a CPU schedule simulator with no model arithmetic; its CPU
        # path for this metric is the oracle port executing the same GPT stage math.  This arm
        # imports neither torch nor the product package.
        if rank != 0:
            return
        smp = LayerSample(args.model)
        for _ in range(args.warmup):
            smp.step()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            smp.step()
            times.append(time.perf_counter() - t0)
        total = sum(times)
        value = smp.flops * args.steps / total / flops_per_token(args.model)
        replay = cpu_schedule_replay()
        cb = {"value": value, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port-extrapolated",
              "sample": smp.describe(args.steps, total)}
        line = {"impl": "reference", "metric": metric, "value": value, "unit": "tokens/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * total / args.steps,
                "step_definition": "one bounded sample (1 layer x 1 sequence forward+backward) of the workload",
                "higher_is_better": True, "dtype": "f32", "data": "synthetic", "config": cfg,
                "cpu_baseline": cb,
                "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "full_schedule_replay": replay,
                "reference_schedule_path": schedule_baseline(),
                "note": "the reference (ppsim) has no model arithmetic; its CPU path for tokens/s is "
                        "the oracle port executing the same GPT stage math"}
        assert "paper_2605_29664_b200" not in sys.modules  # the reference arm never loads libamdp.so
        print(json.dumps(line), flush=True)
        return

    model = model_cfg(args.model)
    model.recompute = bool(args.recompute)

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    from paper_2605_29664_b200 import engine as E
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.comm == "nccl":
            obj = [E.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return float(t.item())

    windows = max(args.steps, args.warmup)
    opt = E.OptimizerConfig(lr=1e-4, weight_decay=0.0)
    run = E.RunConfig(depth=args.depth, threshold=args.threshold, windows=windows, optimizer=opt, schedule=args.schedule,
                      zero=zero, world_size=world, rank=rank, comm=args.comm)
    eng = E.Engine(model, run, nccl_id, allgather=E.torch_allgather() if world > 1 else None)
    M = run.num_minibatches
    toks = E.PinnedTokens(M, model.tokens_per_minibatch)
    E.synthetic_tokens(model, run.data_seed, 0, M, out=toks)
    losses = toks.losses  # pinned: runs over pinned buffers are CUDA graphs (one GPU)
    if args.no_graphs:
        eng.set_graphs(False)

    # warm-up windows (untimed, eager: every lazy initialisation happens here)
    eng.run_windows(args.warmup, toks.inputs, toks.labels, losses)
    # value: tokens resident in HBM
    eng.stage_tokens(toks.inputs, toks.labels)
    # untimed: the timed configuration's CUDA graph is captured on its first run
    eng.run_windows(args.steps, toks.inputs, toks.labels, losses, resident=True)
    barrier()
    with ClockSampler(local) as clk:
        eng.run_windows(args.steps, toks.inputs, toks.labels, losses, resident=True)
        barrier()
    st = eng.stats()
    dev_ms = max_over_ranks(st["device_ms"])
    host_issue_ms = max_over_ranks(st["host_issue_ms"])
    value = args.steps * tok_step / (dev_ms / 1e3)
    tl = eng.timeline()
    launches = int(sum_over_ranks(st["kernels_launched"]))
    busy_frac = st["busy_ms"] / st["device_ms"] if st["device_ms"] else None
    try:
        from paper_2605_29664_b200 import ppsim as P
        logical_bubble = float(P.bubble_ratio(tl, 1)) if args.steps > 2 else float(P.bubble_ratio(tl, 0))
    except Exception:
        logical_bubble = None
    phys_bubble = max_over_ranks(1.0 - busy_frac) if busy_frac is not None else None
    # e2e through the public API with pinned host buffers (its graph captured untimed first)
    eng.run_windows(args.steps, toks.inputs, toks.labels, losses, resident=False)
    barrier()
    t0 = time.perf_counter()
    eng.run_windows(args.steps, toks.inputs, toks.labels, losses, resident=False)
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    st2 = eng.stats()
    e2e = args.steps * tok_step / e2e_s

    projection = None
    if world == 1 and args.steps > 2:
        try:  # d-GPU projection (static-order replay, reference bubble_ratio) from per-task costs
            # measured on the serial executor: with concurrent compute streams the tasks of
            # different logical devices overlap, so their event spans are not their own costs
            from paper_2605_29664_b200 import projection as PR
            ns = eng.plan()["compute_streams"]
            eng.set_streams(1)
            eng.run_windows(args.steps, toks.inputs, toks.labels, losses, resident=True)  # untimed
            tl = eng.timeline()
            lanes = eng.lane_events()
            eng.set_streams(ns)
            gap_ns = model.tokens_per_minibatch * model.hidden * 2 / 770e9 * 1e9
            numel = [lib_numel(eng, i) for i in range(args.depth)]
            pol = E.RunConfig(depth=args.depth, threshold=args.threshold, windows=args.steps,
                              schedule=args.schedule, zero=zero).policy()
            part = eng.plan()["partition"]
            segs = [part[i] + (i == 0) + (i == args.depth - 1) for i in range(args.depth)]
            projection = PR.project(tl, args.depth, args.threshold, args.steps, model.tokens_per_minibatch, gap_ns,
                                    stage_numel=numel, policy=pol, lane_events=lanes, segments=segs)
            if args.schedule == "AMDP" and zero:
                # the same measured costs under AMDP's other update mode: replicated weights,
                # window gradient all-reduced over the stage's devices, every replica stepping
                # its own optimizer (an Update costs the measured fused optimizer step + the
                # all-reduce), builder.hpp:306-336
                alt = E.RunConfig(depth=args.depth, threshold=args.threshold, windows=args.steps,
                                  schedule="AMDP", zero=False).policy()
                pa = PR.project(tl, args.depth, args.threshold, args.steps, model.tokens_per_minibatch, gap_ns,
                                stage_numel=numel, policy=alt, lane_events=lanes)
                projection["allreduce_update_variant"] = {k: pa[k] for k in
                                                          ("bubble", "bubble_without_collectives", "tokens_per_s")}
        except Exception as e:  # never let the projection break the bench line
            projection = {"error": str(e)[:200]}


    # per-kernel-class timing for the roofline
    kern = {}
    if not args.no_kernel_timing:
        eng.set_kernel_timing(True)
        barrier()
        eng.run_windows(min(args.steps, 2), toks.inputs, toks.labels, losses, resident=True)
        barrier()
        kern = eng.kernel_stats()
        eng.set_kernel_timing(False)

    pk, src = peaks()
    gem = [kern.get(c, {}) for c in ("gemm_fwd", "gemm_dgrad", "gemm_wgrad")]
    g_ms = sum(k.get("ms", 0) for k in gem)
    g_fl = sum(k.get("flops", 0) for k in gem)
    g_n = sum(k.get("launches", 0) for k in gem)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    achieved = (g_fl / (g_ms / 1e3) / 1e12) if g_ms else None
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    roofline = {"kernel": "gemm_bf16_tcgen05 (all stage GEMMs)", "bound": "tensor",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": f"{src} bf16_tflops_sustained (kernel inside a long step)",
                "launches": g_n, "avg_launch_us": (1e3 * g_ms / g_n) if g_n else None,
                "share_of_step": (g_ms / sum(k["ms"] for k in kern.values())) if kern else None}
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                   "tflops": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1) if v["flops"] and v["ms"] else None,
                   "gbs": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["bytes"] and v["ms"] else None}
               for k, v in kern.items()}
    # MFU against the dense bf16 spec peak (2.25 PF/s per B200); the ratio to the measured,
    # power-capped sustained cuBLAS rate on this box is reported beside it
    mfu = value * model.flops_per_token() / (args.gpus * SPEC_BF16_TFLOPS * 1e12)
    mfu_sustained = value * model.flops_per_token() / (args.gpus * peak * 1e12)

    line = {"metric": metric, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (arithmetic-progression token streams, random-init weights)",
            "config": cfg,
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": st2["h2d_bytes"] // args.steps,
                    "d2h_bytes_per_step": st2["d2h_bytes"] // args.steps},
            "gpu_launches": launches,
            "cuda_graph": bool(st.get("graph_replayed")),
            "host_issue_ms_per_step": host_issue_ms / args.steps,
            "roofline": roofline,
            "model_flops_utilization": mfu,
            "model_flops_vs_measured_sustained_peak": mfu_sustained,
            "bubble": {"physical_gpu": phys_bubble, "logical_devices_bubble_ratio_w1": logical_bubble,
                       f"projected_d{args.depth}_gpus": projection},
            "kernels": kernels,
            "memory_gb": {k: (round(v / 1e9, 3) if not k.endswith(("_units", "_slots")) else v)
                          for k, v in eng.plan()["memory"].items()},
            "clocks": clk.summary()}
    if rank == 0:
        if world == 1:
            line["cpu_baseline"] = {k: v for k, v in cpu_port_baseline(args.model).items() if k != "cpu_gflops"}
            line["cpu_baseline"]["full_schedule_replay"] = cpu_schedule_replay()
            sb = schedule_baseline()
            if sb:
                line["reference_schedule_path"] = sb
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
