"""Mean measured Forward / Backward task durations per stage from the bench workload's
device timeline (record_events), for comparing two library builds on one box (AMDP_LIB)."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_29664_b200 import engine as E
model = E.ModelConfig.gpt_1p3b()
run = E.RunConfig(depth=8, threshold=32, windows=4, optimizer=E.OptimizerConfig(lr=1e-4, weight_decay=0.0))
eng = E.Engine(model, run)
M = run.num_minibatches
toks = E.PinnedTokens(M, model.tokens_per_minibatch)
E.synthetic_tokens(model, run.data_seed, 0, M, out=toks)
losses = np.zeros(M, np.float32)
eng.run_windows(2, toks.inputs, toks.labels, losses)
eng.stage_tokens(toks.inputs, toks.labels)
eng.run_windows(4, toks.inputs, toks.labels, losses, resident=True)
tl = eng.timeline()
d = {}
for dev in tl.per_device:
    for ev in dev:
        if ev.window < 1:
            continue
        k = (ev.kind.name[0], ev.stage)
        d.setdefault(k, []).append(float(ev.duration) / 1e6)
out = {f"{k[0]}{k[1]}": round(statistics.mean(v), 3) for k, v in sorted(d.items()) if k[0] in "FB"}
out["device_ms_per_window"] = eng.stats()["device_ms"] / 4
print(json.dumps(out))
eng.close()
