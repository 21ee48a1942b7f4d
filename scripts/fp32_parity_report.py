"""Observed engine-vs-oracle errors of the bf16 production path and the fp32 validation mode
on the same run (tiny GPT and a head_dim-64 model, AMDP D=4 ZeRO, AdamW, 3 windows): max
per-minibatch loss error and final-weight errors, each mode against the oracle replaying the
reference trace with (bf16) or without (fp32) bf16 rounding emulation.

    python scripts/fp32_parity_report.py > profiles/r02/fp32_validation.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import gpt_oracle as O
    from paper_2605_29664_b200 import engine as E
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "sched_golden.json")))
    trace = next(e["csv"] for e in gold if e["config"] == ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 24, 1] and "csv" in e)
    out = {}
    for name, dims in (("tiny", (4, 128, 4, 512, 1024, 64)), ("hd64", (4, 512, 8, 2048, 2048, 256))):
        for fp32 in (False, True):
            m = E.ModelConfig(*dims)
            m.layers_per_stage = [1, 1, 1, 1]
            m.fp32_validation = fp32
            run = E.RunConfig(depth=4, threshold=8, windows=3,
                              optimizer=E.OptimizerConfig(kind=3, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                                                          weight_decay=0.0))
            eng = E.Engine(m, run)
            init = [eng.stage_params(i) for i in range(4)]
            inputs, labels = E.synthetic_tokens(m, run.data_seed, 0, run.num_minibatches)
            losses = eng.run(inputs, labels)
            om = O.Model(*dims, 4, True, m.seed)
            ol, om_, _ = O.replay(trace, om, [1, 1, 1, 1], O.Opt("adamw", 1e-3, 0.9, 0.95, 1e-8, 0.0), 8, inputs,
                                  labels, emulate_bf16=not fp32)
            plan = eng.plan()
            werr, uerr = [], []
            for i in range(4):
                st = plan["stages"][i]
                ref = O.flat_stage(om_[i], st["params"], st["numel"])
                got = eng.stage_params(i).astype(np.float64)
                werr.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
                uerr.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref - init[i])))
            out[f"{name}_{'fp32' if fp32 else 'bf16'}"] = {
                "loss_max_rel_err": float(np.max(np.abs(losses - ol) / np.abs(ol))),
                "weights_max_rel_err": max(werr), "weights_err_over_update": max(uerr)}
            eng.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
