import sys, os, math, torch
sys.path.insert(0, "/root/repo")
from paper_2605_29664_b200 import kernels as K
def ref(qkv, B, S, H, D, causal):
    q, k, v = qkv.float().view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    s = q @ k.transpose(-1, -2) / math.sqrt(D)
    if causal:
        s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device=qkv.device).triu(1), float("-inf"))
    return (s.softmax(-1) @ v).permute(0, 2, 1, 3).reshape(B * S, H * D)
for (B, S, H, D, c) in [(2, 512, 3, 80, True), (2, 512, 3, 80, False), (1, 2048, 2, 80, True), (2, 512, 3, 128, True)]:
    torch.manual_seed(3)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, S, H, D, c)
    x = qkv.float().requires_grad_()
    r = ref(x, B, S, H, D, c); r.backward(dout.float())
    dq = K.attention_bwd(qkv, out, dout, lse, B, S, H, D, c)
    torch.cuda.synchronize()
    rel = lambda a, b: ((a.double() - b.double()).norm() / b.double().norm()).item()
    g = x.grad; hd = H * D
    print((B, S, H, D, c), "out", round(rel(out, r), 5), [round(rel(dq[:, p*hd:(p+1)*hd], g[:, p*hd:(p+1)*hd]), 5) for p in range(3)])
    if D == 80:
        e = (dq[:, :hd].float() - g[:, :hd]).abs().view(B * S, H, D).amax(dim=(0, 1))
        print("  dq max err per dim (first 8, 60-80):", [round(v, 3) for v in e[:8].tolist()], [round(v, 3) for v in e[60:80].tolist()])
        e = (dq[:, hd:2*hd].float() - g[:, hd:2*hd]).abs().view(B * S, H, D).amax(dim=(0, 1))
        print("  dk max err per dim (60-80):", [round(v, 3) for v in e[60:80].tolist()])
