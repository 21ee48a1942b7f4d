import sys, os, torch, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K
T, h = 8192, 2048
x = torch.randn(T, h, device="cuda").bfloat16(); dy = torch.randn(T, h, device="cuda").bfloat16()
rg = torch.randn(T, h, device="cuda").bfloat16()
g = torch.ones(h, device="cuda"); b = torch.zeros(h, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
def med(fn, n=20):
    ts = []
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)
y, mean, rstd = K.layernorm_fwd(x, g, b)
dg = torch.zeros(h, device="cuda"); db = torch.zeros(h, device="cuda")
f = med(lambda: K.layernorm_fwd(x, g, b))
bw = med(lambda: K.layernorm_bwd(dy, x, g, mean, rstd, rg, dg, db))
print(json.dumps({"ln_fwd_us": f * 1e3, "ln_fwd_gbs": 4 * T * h / f / 1e6, "ln_bwd_us": bw * 1e3,
                  "ln_bwd_gbs": (8 + 4) * T * h / bw / 1e6}))
