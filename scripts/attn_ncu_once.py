"""One forward + one backward of the tensor-core attention at each model shape (for an ncu
capture: `ncu --set full -k regex:fa_ ... python scripts/attn_ncu_once.py`)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K  # noqa: E402

SHAPES = [(4, 512, 16, 64, False), (4, 1024, 16, 64, True), (4, 2048, 16, 128, True), (4, 2048, 32, 80, True)]
for B, S, H, D, causal in SHAPES:
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, S, H, D, causal)
    K.attention_bwd(qkv, out, dout, lse, B, S, H, D, causal)
    torch.cuda.synchronize()
