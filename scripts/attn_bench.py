"""Attention kernels at the 1.3B shape: median of 20 timed runs each (CUDA events)."""
import sys, os, json, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K
B, S, H, D = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 2048, 16, 128))]
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, S, H, D)
def med(fn, n=20):
    ts = []
    for _ in range(3): fn()
    for _ in range(n):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)
fl = 4.0 * B * H * S * S * D / 2
f = med(lambda: K.attention_fwd(qkv, B, S, H, D))
b = med(lambda: K.attention_bwd(qkv, out, dout, lse, B, S, H, D))
q, k, v = qkv.view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
sd = med(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True))
qq, kk, vv = [t.detach().clone().requires_grad_() for t in (q, k, v)]
o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
g = torch.randn_like(o)
sdb = med(lambda: torch.autograd.grad(o, (qq, kk, vv), g, retain_graph=True))
print(json.dumps({"fwd_ms": f, "fwd_tflops": fl / f / 1e9, "bwd_ms": b, "bwd_tflops": 2.5 * fl / b / 1e9,
                  "sdpa_fwd_ms": sd, "sdpa_bwd_ms": sdb}))
