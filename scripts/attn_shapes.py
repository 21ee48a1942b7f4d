"""Attention forward / backward at the model shapes, back-to-back launches (per-launch time of
20 consecutive calls, median of 10), next to torch SDPA (cuDNN / flash backends) on the same
tensors.  FLOPs: 4 B H S^2 D forward (halved when causal), 2.5x that backward.

    python scripts/attn_shapes.py            -> one JSON line per shape
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K  # noqa: E402


def per_call(fn, n=10, reps=20):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / reps)
    return statistics.median(ts)


SHAPES = [  # name, B, S, H, D, causal
    ("bert_large", 4, 512, 16, 64, False),
    ("gpt_350m", 4, 1024, 16, 64, True),
    ("gpt_1p3b", 4, 2048, 16, 128, True),
    ("gpt_2p7b", 4, 2048, 32, 80, True),
]
only = set(sys.argv[1:])
for name, B, S, H, D, causal in SHAPES:
    if only and name not in only:
        continue
    torch.manual_seed(0)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, S, H, D, causal)
    fl = 4.0 * B * H * S * S * D / (2 if causal else 1)
    f = per_call(lambda: K.attention_fwd(qkv, B, S, H, D, causal))
    b = per_call(lambda: K.attention_bwd(qkv, out, dout, lse, B, S, H, D, causal))
    # the engine's call: delta supplied (dO GEMM epilogue); dQ from stored dS^T vs recomputed
    delta = (dout.float() * out.float()).view(B, S, H, D).sum(-1).permute(0, 2, 1).contiguous()
    bd = per_call(lambda: K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, causal))
    br = per_call(lambda: K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, causal, scratch=False))
    q, k, v = [t.contiguous() for t in qkv.view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)]
    sd = per_call(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal))
    qq, kk, vv = [t.detach().clone().requires_grad_() for t in (q, k, v)]
    o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=causal)
    g = torch.randn_like(o)
    sdb = per_call(lambda: torch.autograd.grad(o, (qq, kk, vv), g, retain_graph=True))
    print(json.dumps({"shape": name, "B": B, "S": S, "H": H, "D": D, "causal": causal,
                      "fwd_us": round(1e3 * f, 2), "fwd_tflops": round(fl / f / 1e9, 1),
                      "bwd_us": round(1e3 * b, 2), "bwd_tflops": round(2.5 * fl / b / 1e9, 1),
                      "bwd_delta_us": round(1e3 * bd, 2), "bwd_delta_tflops": round(2.5 * fl / bd / 1e9, 1),
                      "bwd_delta_recompute_dq_us": round(1e3 * br, 2),
                      "sdpa_fwd_us": round(1e3 * sd, 2), "sdpa_bwd_us": round(1e3 * sdb, 2)}), flush=True)
