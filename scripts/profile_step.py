"""One short AMDP window for ncu launch lists / captures (never a bench number).  Weight init
and a first warm-up window run outside the profiled range (ncu --profile-from-start off).
    python scripts/profile_step.py [model depth threshold]   (default: 1p3b 8 32)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_29664_b200 import engine as E
name, depth, thr = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else ("1p3b", 8, 32)
model = {"1p3b": E.ModelConfig.gpt_1p3b, "350m": E.ModelConfig.gpt_350m, "2p7b": E.ModelConfig.gpt_2p7b,
         "bert": E.ModelConfig.bert_large}[name]()
run = E.RunConfig(depth=depth, threshold=thr, windows=1, record_events=False)
eng = E.Engine(model, run)
inp, lab = E.synthetic_tokens(model, run.data_seed, 0, run.num_minibatches)
eng.run(inp, lab)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.run(inp, lab)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
