import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K
B, S, H, D = 4, 2048, 16, 128
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
for _ in range(3):
    out, lse = K.attention_fwd(qkv, B, S, H, D)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
for SS in (2048, 2112):
    q2 = torch.randn(B * SS, 3 * H * D, device="cuda").bfloat16()
    K.attention_fwd(q2, B, SS, H, D); torch.cuda.synchronize()
    s.record()
    for _ in range(10): K.attention_fwd(q2, B, SS, H, D)
    e.record(); torch.cuda.synchronize()
    print(SS, s.elapsed_time(e) / 10, "ms")
