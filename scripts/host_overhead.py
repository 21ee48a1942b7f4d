"""Host-side cost of issuing the library's kernels (what bounds the small models: BERT-large
D=8 issues ~17k launches per window).  Times N back-to-back calls of each C-ABI entry point on
tiny shapes (the GPU keeps up, so the host loop is what is measured), against a ctypes no-op.

    python scripts/host_overhead.py            -> one JSON line, microseconds per call
"""
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_29664_b200 import _native as N  # noqa: E402


def per_call(fn, n=400):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    return 1e6 * dt / n


def main():
    torch.cuda.set_device(0)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    out = {}
    out["ctypes_noop"] = per_call(lambda: N.lib.amdp_version())
    M = Nn = K = 256
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(Nn, K, device="cuda").bfloat16()
    C = torch.empty(M, Nn, device="cuda").bfloat16()
    args = N.GemmArgs(M, Nn, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), Nn, 0, 0, 0, 0, 0, 1.0, 0, 0, 0)
    out["gemm_256"] = per_call(lambda: N.lib.amdp_gemm(ctypes.byref(args), s))
    M2 = 2048
    A2 = torch.randn(M2, 1024, device="cuda").bfloat16()
    B2 = torch.randn(1024, 1024, device="cuda").bfloat16()
    C2 = torch.empty(M2, 1024, device="cuda").bfloat16()
    args2 = N.GemmArgs(M2, 1024, 1024, A2.data_ptr(), 1024, 0, B2.data_ptr(), 1024, 0, C2.data_ptr(), 1024, 0, 0, 0, 0,
                       0, 1.0, 0, 0, 0)
    out["gemm_bert_out_proj"] = per_call(lambda: N.lib.amdp_gemm(ctypes.byref(args2), s), n=200)
    x = torch.randn(256, 1024, device="cuda").bfloat16()
    g = torch.ones(1024, device="cuda")
    b = torch.zeros(1024, device="cuda")
    y = torch.empty_like(x)
    mu = torch.empty(256, device="cuda")
    rs = torch.empty(256, device="cuda")
    out["layernorm_fwd"] = per_call(lambda: N.lib.amdp_layernorm_fwd(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(b.data_ptr()),
        ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(mu.data_ptr()), ctypes.c_void_p(rs.data_ptr()), 256, 1024,
        ctypes.c_float(1e-5), s))
    qkv = torch.randn(512, 3 * 1024, device="cuda").bfloat16()
    o = torch.empty(512, 1024, device="cuda").bfloat16()
    lse = torch.empty(16 * 512, device="cuda")
    out["attention_fwd_s512"] = per_call(lambda: N.lib.amdp_attention_fwd(
        ctypes.c_void_p(qkv.data_ptr()), ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(lse.data_ptr()), 1, 512, 16, 64,
        1, None, s), n=200)
    ev = torch.cuda.Event()
    out["torch_event_record"] = per_call(lambda: ev.record())
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
