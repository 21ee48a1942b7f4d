"""One short 1.3B AMDP run for ncu launch lists / captures (never a bench number).  Weight init
and a first warm-up window run outside the profiled range (ncu --profile-from-start off)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_29664_b200 import engine as E
model = E.ModelConfig.gpt_1p3b()
run = E.RunConfig(depth=8, threshold=32, windows=1, record_events=False)
eng = E.Engine(model, run)
inp, lab = E.synthetic_tokens(model, run.data_seed, 0, run.num_minibatches)
eng.run(inp, lab)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.run(inp, lab)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
