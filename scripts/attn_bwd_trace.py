"""Per-phase clock64 trace of CTA 0 of the tcgen05 dQ kernel (AMDP_ATTN_DQ=recompute) and of
the dK/dV kernel (times relative to its first recorded event)."""
import sys, os, ctypes, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K, _native as N
N.lib.amdp_debug_attention_bwd_trace.argtypes = [ctypes.c_void_p]
B, S, H, D = 4, 2048, 16, 128
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, S, H, D)
for _ in range(3): K.attention_bwd(qkv, out, dout, lse, B, S, H, D)
buf = torch.zeros(32 * 64, dtype=torch.int64, device="cuda")
N.lib.amdp_debug_attention_bwd_trace(ctypes.c_void_p(buf.data_ptr()))
K.attention_bwd(qkv, out, dout, lse, B, S, H, D); torch.cuda.synchronize()
N.lib.amdp_debug_attention_bwd_trace(None)
t = buf.view(32, 64).cpu(); t0 = int(t[7, 0])
names = ["mma:kv_full", "mma:s_empty(S iss)", "mma:p_full(dQ iss)", "wg:s_full", "wg:computed", "wg:arrived", "prod:kv_empty",
         "-", "mma:S issued", "mma:dQ issued"]
print("n  " + " ".join(f"{x:>12s}" for i, x in enumerate(names) if i != 7))
for n in range(32):
    print(f"{n:2d} " + " ".join(f"{int(t[s, n]) - t0 if t[s, n] else -1:12d}" for s in range(10) if s != 7))

d = t[16:24, :]
t0 = int(d[d > 0].min()) if (d > 0).any() else t0
names = ["mma:u_full", "mma:S issued", "mma:p_full", "mma:dVdK issued", "wgA:s_full", "wgA:computed", "prod:u_empty", "wgA:arrived"]
print("dK/dV kernel CTA 0 (kt = 0), per 64-query half unit u (softmax columns: warpgroup A only)")
print("n  " + " ".join(f"{x:>14s}" for x in names))
for n in range(24):
    print(f"{n:2d} " + " ".join(f"{int(t[16 + s, n]) - t0 if t[16 + s, n] else -1:14d}" for s in range(8)))
