"""Which library calls can be captured into a CUDA graph?  Captures each on a fresh stream
(relaxed mode) and reports success / the CUDA error, e.g.
    python scripts/probes/graph_probe.py
"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2605_29664_b200 import _native as N  # noqa: E402

cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None


def capture(name, fn, res):
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            fn(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        g.replay()
        torch.cuda.synchronize()
        res[name] = "ok"
    except Exception as e:  # noqa: BLE001
        res[name] = str(e)[:200]
        torch.cuda.synchronize()


def main():
    torch.cuda.set_device(0)
    res = {}
    x = torch.randn(256, 1024, device="cuda").bfloat16()
    g = torch.ones(1024, device="cuda")
    b = torch.zeros(1024, device="cuda")
    y = torch.empty_like(x)
    mu = torch.empty(256, device="cuda")
    rs = torch.empty(256, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def ln(s):
        N.check(N.lib.amdp_layernorm_fwd(P(x), P(g), P(b), P(y), P(mu), P(rs), 256, 1024, ctypes.c_float(1e-5), s), "ln")
    # warm (lazy attributes) outside capture
    ln(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    capture("layernorm_fwd (PDL launch first in graph)", ln, res)

    def ln_after_kernel(s):
        y.zero_()
        ln(s)
    capture("torch kernel then PDL layernorm", ln_after_kernel, res)

    def ln_after_memset(s):
        mu.fill_(0)
        ln(s)
    capture("memset then PDL", ln_after_memset, res)

    M = 512
    A = torch.randn(M, 1024, device="cuda").bfloat16()
    B = torch.randn(1024, 1024, device="cuda").bfloat16()
    C = torch.empty(M, 1024, device="cuda").bfloat16()
    args = N.GemmArgs(M, 1024, 1024, A.data_ptr(), 1024, 0, B.data_ptr(), 1024, 0, C.data_ptr(), 1024, 0, 0, 0, 0, 0,
                      1.0, 0, 0, 0)

    def gemm(s):
        N.check(N.lib.amdp_gemm(ctypes.byref(args), s), "gemm")
    gemm(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    capture("gemm pair (cluster + PDL)", gemm, res)
    capture("gemm after layernorm", lambda s: (ln(s), gemm(s)), res)
    qkv = torch.randn(512, 3 * 1024, device="cuda").bfloat16()
    o = torch.empty(512, 1024, device="cuda").bfloat16()
    lse = torch.empty(16 * 512, device="cuda")

    def attn(s):
        N.check(N.lib.amdp_attention_fwd(P(qkv), P(o), P(lse), 1, 512, 16, 64, 1, s), "attn")
    attn(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    capture("attention fwd tcgen05", attn, res)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
