"""Per-CTA start/end (globaltimer) of the tensor-core attention forward: wave structure,
per-CTA duration vs its KV-block count, SM idle time."""
import sys, os, ctypes, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K, _native as N
N.lib.amdp_debug_attention_cta_times.argtypes = [ctypes.c_void_p]
B, S, H, D = [int(v) for v in sys.argv[1:5]] if len(sys.argv) > 4 else (4, 2048, 16, 128)
CAUSAL = bool(int(sys.argv[5])) if len(sys.argv) > 5 else True
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
for _ in range(3): K.attention_fwd(qkv, B, S, H, D, CAUSAL)
n_qt = S // 256
ncta = min(n_qt * H * B, torch.cuda.get_device_properties(0).multi_processor_count)
buf = torch.zeros(3 * ncta, dtype=torch.int64, device="cuda")
N.lib.amdp_debug_attention_cta_times(ctypes.c_void_p(buf.data_ptr()))
K.attention_fwd(qkv, B, S, H, D, CAUSAL); torch.cuda.synchronize()
N.lib.amdp_debug_attention_cta_times(None)
t = buf.view(ncta, 3).cpu()
t0 = int(t[:, 0].min()); t1 = int(t[:, 1].max())
d = sorted(int(t[i, 1] - t[i, 0]) for i in range(ncta))
st = sorted(int(t[i, 0]) - t0 for i in range(ncta))
print(f"kernel span {(t1 - t0) / 1e3:.1f} us, {ncta} persistent CTAs; CTA busy us min {d[0] / 1e3:.1f} "
      f"median {d[len(d) // 2] / 1e3:.1f} max {d[-1] / 1e3:.1f}; start skew max {st[-1] / 1e3:.1f} us")
