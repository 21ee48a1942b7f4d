import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K
B, S, H, D = 4, 2048, 16, 128
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, S, H, D)
for _ in range(3):
    K.attention_bwd(qkv, out, dout, lse, B, S, H, D)
torch.cuda.synchronize()
