"""One backward per dQ variant (stored dS^T + dQ GEMM vs recomputing dQ kernel) at a model
shape, for an ncu launch list:  python scripts/attn_dq_probe.py B S H D causal"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K  # noqa: E402

B, S, H, D, causal = (int(a) for a in sys.argv[1:6])
torch.manual_seed(0)
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, S, H, D, bool(causal))
delta = (dout.float() * out.float()).view(B, S, H, D).sum(-1).permute(0, 2, 1).contiguous()
for _ in range(2):
    K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, bool(causal))
    K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, bool(causal), scratch=False)
torch.cuda.synchronize()
