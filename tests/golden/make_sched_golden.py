"""Generates tests/golden/sched_golden.json from the UNMODIFIED reference, compiled in place
by oracle/Makefile into oracle/_ref/ppsim_ref.  Run here (the container that has
/root/reference); the fixture is committed so the GPU box and CI never need the reference.

    make -C oracle _ref/ppsim_ref && python tests/golden/make_sched_golden.py
"""
import hashlib
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "ppsim_ref")

# (policy, depth, devices, fwd, bwd, update, comm, inj, pipes, thr, M, zero)
CONFIGS = []
for d in (2, 4, 8):
    P = d // 2
    for tb in ("1", "2", "3/2", "3"):
        for zero in (1, 0):
            for thr_mul in (1, 2, 4):
                thr = max(2 * P, thr_mul * d)
                CONFIGS.append(("AMDP", d, d, "1", tb, "0", "0", 2, P, thr, 4 * thr, zero))
CONFIGS += [
    ("AMDP", 8, 8, "1", "2", "0", "0", 2, 4, 32, 512, 1),   # the canonical manifest
    ("AMDP", 8, 8, "1", "1", "0", "0", 2, 4, 32, 512, 1),
    ("AMDP", 4, 4, "1", "2", "0", "0", 2, 2, 8, 32, 1),     # tiny GPT config
    ("AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 1),
    ("AMDP", 2, 2, "1", "2", "0", "0", 2, 1, 4, 64, 1),
    ("AMDP", 4, 4, "1", "2", "0", "1/2", 2, 2, 8, 32, 1),   # comm gap changes the order
    ("AMDP", 8, 8, "1", "2", "1/4", "1/10", 2, 4, 16, 64, 1),
    ("AMDP", 6, 6, "2,1,1,1,1,3", "4,2,2,2,2,5", "1", "0", 2, 3, 6, 24, 0),
    ("AMDP", 16, 16, "1", "2", "0", "0", 2, 8, 32, 128, 1),
    ("DAPPLE", 4, 4, "1", "2", "0", "1/2", 8, 1, 8, 8, 0),
    ("DAPPLE", 8, 8, "1", "2", "0", "0", 8, 1, 8, 32, 0),
    ("GPipe", 4, 4, "1", "2", "0", "0", 4, 1, 4, 16, 0),
    ("Interleaved1F1B", 8, 4, "1", "2", "0", "0", 4, 1, 4, 16, 0),
    ("Chimera", 4, 4, "1", "2", "0", "0", 4, 2, 4, 16, 0),
    ("Chimera", 8, 8, "1", "1", "0", "0", 8, 2, 8, 16, 0),
    ("PipeDreamAsync", 4, 4, "1", "1", "0", "0", 2, 1, 1, 16, 0),
    ("PipeDreamAsync", 8, 8, "1", "2", "1/2", "0", 8, 1, 4, 32, 0),
    ("DAPPLE", 4, 4, "1", "1", "0", "0", 8, 1, 8, 32, 0),     # tiny GPT on the executor (P = 1)
    ("GPipe", 4, 4, "1", "1", "0", "0", 8, 1, 8, 32, 0),
    ("Chimera", 4, 4, "1", "1", "0", "0", 8, 2, 8, 32, 0),            # replicated, two pipelines
    ("Interleaved1F1B", 4, 2, "1", "1", "0", "0", 8, 1, 8, 32, 0),    # two chunks per device
    ("PipeDreamAsync", 4, 4, "1", "1", "0", "0", 4, 1, 8, 32, 0),     # update per backward
]
# Production-shaped engine-vs-oracle parity runs (tests/test_parity_prod_gpu.py): the trace is
# stored for each (declared 1:1 -> preload 1; declared 1:2 -> preload 2, the reference's
# canonical manifests/amdp_d8.json cost model), ZeRO and replicated.
PARITY = [
    ("AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 24, 1),
    ("AMDP", 4, 4, "1", "2", "0", "0", 2, 2, 8, 24, 0),
    ("AMDP", 8, 8, "1", "2", "0", "0", 2, 4, 16, 32, 1),
    ("AMDP", 8, 8, "1", "1", "0", "0", 2, 4, 16, 32, 0),
]
CONFIGS += PARITY


def run(cfg, mode):
    args = [REF] + [str(x) for x in cfg] + [mode, "1"]
    return subprocess.run(args, check=True, capture_output=True, text=True).stdout


def main():
    out = []
    for cfg in CONFIGS:
        csv = run(cfg, "csv")
        if csv.startswith("ERROR"):
            raise SystemExit(f"{cfg}: {csv}")
        summ = json.loads(run(cfg, "summary"))
        entry = {"config": list(cfg), "sha256": hashlib.sha256(csv.encode()).hexdigest(),
                 "events": csv.count("\n") - 1, "makespan": summ["makespan"],
                 "bubble_w1": summ["bubble_ratio"], "bubble_w0": summ["bubble_w0"],
                 "max_mismatch": max((e["updates_between"] for e in summ["mismatch"]["entries"]), default=0),
                 "mismatch_nonzero": [[e["stage"], e["minibatch"], e["updates_between"]]
                                      for e in summ["mismatch"]["entries"] if e["updates_between"]],
                 "windows": summ["windows"], "memory": summ["memory"]}
        if (cfg[1] <= 4 and cfg[10] <= 32) or cfg in PARITY:
            entry["csv"] = csv
        out.append(entry)
    with open(os.path.join(HERE, "sched_golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {len(out)} configs")


if __name__ == "__main__":
    main()
