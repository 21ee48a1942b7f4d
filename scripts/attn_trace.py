"""Per-phase clock64 trace of CTA 0 (heaviest 256-query pair tile) of the tcgen05 attention forward."""
import sys, os, ctypes, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K, _native as N
N.lib.amdp_debug_attention_trace.argtypes = [ctypes.c_void_p]
B, S, H, D = [int(v) for v in sys.argv[1:5]] if len(sys.argv) > 4 else (4, 2048, 16, 128)
CAUSAL = bool(int(sys.argv[5])) if len(sys.argv) > 5 else True
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
for _ in range(3): K.attention_fwd(qkv, B, S, H, D, CAUSAL)
buf = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
N.lib.amdp_debug_attention_trace(ctypes.c_void_p(buf.data_ptr()))
K.attention_fwd(qkv, B, S, H, D, CAUSAL); torch.cuda.synchronize()
N.lib.amdp_debug_attention_trace(None)
t = buf.view(16, 64).cpu()
t0 = int(t[10, 0])
names = ["mma:k_full", "wgA:p_full", "wgB:p_full", "mma:PV_A issue", "mma:PV_B issue", "wgA:s_full", "wgB:s_full",
         "-", "prod:k_empty", "prod:v_empty", "start", "wgA:ld_done", "wgA:max_done", "wgA:p_done"]
print("j " + " ".join(f"{n:>14s}" for i, n in enumerate(names) if i != 10))
for j in range(16):
    print(f"{j:2d} " + " ".join(f"{int(t[s, j]) - t0 if t[s, j] else -1:14d}" for s in range(14) if s != 10))
