"""LayerNorm fwd/bwd at the 1.3B shape (T=8192, h=2048; or argv T h), L2 flushed before every launch,
next to a plain torch copy of the same bytes (the practical floor for this size)."""
import sys, os, torch, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K
T, h = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8192, 2048)
x = torch.randn(T, h, device="cuda").bfloat16(); dy = torch.randn(T, h, device="cuda").bfloat16()
rg = torch.randn(T, h, device="cuda").bfloat16()
g = torch.ones(h, device="cuda"); b = torch.zeros(h, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
def med(fn, n=20, do_flush=True):
    ts = []
    for _ in range(n):
        if do_flush:
            flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)
y, mean, rstd = K.layernorm_fwd(x, g, b)
dg = torch.zeros(h, device="cuda"); db = torch.zeros(h, device="cuda")
out = {}
for fl in (True, False):
    tag = "" if fl else "_warm"
    f = med(lambda: K.layernorm_fwd(x, g, b), do_flush=fl)
    bw = med(lambda: K.layernorm_bwd(dy, x, g, mean, rstd, rg, dg, db), do_flush=fl)
    cp = med(lambda: y.copy_(x), do_flush=fl)
    out.update({"ln_fwd_us" + tag: f * 1e3, "ln_fwd_gbs" + tag: 4 * T * h / f / 1e6,
                "ln_bwd_us" + tag: bw * 1e3, "ln_bwd_gbs" + tag: 8 * T * h / bw / 1e6,
                "copy_us" + tag: cp * 1e3, "copy_gbs" + tag: 4 * T * h / cp / 1e6})
# 20 back-to-back launches (no flush): per-launch cost inside a stream
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(20):
    K.layernorm_fwd(x, g, b)
e.record(); torch.cuda.synchronize()
out["ln_fwd_us_stream"] = s.elapsed_time(e) / 20 * 1e3
s.record()
for _ in range(20):
    K.layernorm_bwd(dy, x, g, mean, rstd, rg, dg, db)
e.record(); torch.cuda.synchronize()
out["ln_bwd_us_stream"] = s.elapsed_time(e) / 20 * 1e3
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
