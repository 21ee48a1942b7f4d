"""The BERT-large / GPT-350M stage GEMMs (T = 2048 tokens per minibatch, h = 1024): median of
timed launches (CUDA events) of amdp_gemm next to torch.matmul (cuBLAS).  These products are
4-17 GFLOP, i.e. 32-256 output tiles of 128 x 256 on 148 SMs: wave quantisation, not the
tensor pipe, sets their time.  AMDP_GEMM_* knobs are read once per process.

    python scripts/gemm_small.py [T] [h]    -> one JSON line per GEMM
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_29664_b200 import _native as N
from paper_2605_29664_b200 import kernels as K


def med(fn, n=15, warm=10, reps=20):
    """Per-launch time of `reps` back-to-back launches (a lone launch between two events on an
    idle GPU measures launch latency and clock ramp, not the kernel)."""
    for _ in range(warm):
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


T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
h = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
CASES = [  # name, M, N, K, a_mn, b_mn, epilogue
    ("qkv_fwd", T, 3 * h, h, False, False, N.EPI_STORE_BF16),
    ("out_fwd", T, h, h, False, False, N.EPI_RESIDUAL),
    ("fc1_fwd", T, 4 * h, h, False, False, N.EPI_GELU),
    ("fc2_fwd", T, h, 4 * h, False, False, N.EPI_RESIDUAL),
    ("fc2_dgrad", T, 4 * h, h, False, True, N.EPI_GELU_BWD),
    ("fc1_dgrad", T, h, 4 * h, False, True, N.EPI_STORE_BF16),
    ("out_dgrad", T, h, h, False, True, N.EPI_STORE_BF16),
    ("qkv_dgrad", T, h, 3 * h, False, True, N.EPI_STORE_BF16),
    ("fc2_wgrad", h, 4 * h, T, True, True, N.EPI_ACCUM_F32),
    ("fc1_wgrad", 4 * h, h, T, True, True, N.EPI_ACCUM_F32),
    ("out_wgrad", h, h, T, True, True, N.EPI_ACCUM_F32),
    ("qkv_wgrad", 3 * h, h, T, True, True, N.EPI_ACCUM_F32),
]
tot, tot_t = 0.0, 0.0
for name, M, Nn, Kk, a_mn, b_mn, epi in CASES:
    A = torch.randn(Kk, M, device="cuda").bfloat16() if a_mn else torch.randn(M, Kk, device="cuda").bfloat16()
    B = torch.randn(Kk, Nn, device="cuda").bfloat16() if b_mn else torch.randn(Nn, Kk, device="cuda").bfloat16()
    dt = torch.float32 if epi in (N.EPI_ACCUM_F32, N.EPI_STORE_F32) else torch.bfloat16
    C = torch.zeros(M, Nn, dtype=dt, device="cuda")
    extra = {}
    if epi in (N.EPI_GELU_BWD, N.EPI_RESIDUAL):
        extra = dict(aux=torch.randn(M, Nn, device="cuda").bfloat16(), ld_aux=Nn)
    if epi == N.EPI_GELU:
        extra = dict(C2=torch.empty(M, Nn, dtype=torch.bfloat16, device="cuda"), ldc2=Nn)
    ms = med(lambda: K.gemm(A, B, M=M, N_=Nn, K=Kk, a_mn=a_mn, b_mn=b_mn, C=C, epilogue=epi, **extra))
    Al = A.T if a_mn else A
    Bl = B if b_mn else B.T
    ms_t = med(lambda: torch.matmul(Al, Bl))
    fl = 2.0 * M * Nn * Kk
    tot += ms
    tot_t += ms_t
    print(json.dumps(dict(kernel=name, M=M, N=Nn, K=Kk, us=round(1e3 * ms, 2), tflops=round(fl / ms / 1e9, 1),
                          torch_us=round(1e3 * ms_t, 2), torch_tflops=round(fl / ms_t / 1e9, 1))), flush=True)
print(json.dumps(dict(total_us=round(1e3 * tot, 1), torch_total_us=round(1e3 * tot_t, 1),
                      mode=os.environ.get("AMDP_GEMM_MODE", "auto"))))
