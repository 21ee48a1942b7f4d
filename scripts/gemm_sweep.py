"""GEMM variant sweep at the 1.3B stage shapes: median of N timed launches (CUDA events)
for each (shape, operand majors, epilogue), next to torch.matmul (cuBLAS) on the same
logical product.  Environment knobs of amdp_gemm (AMDP_GEMM_STAGES / _TAIL / _MODE) are
read once per process, so run one process per setting."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_29664_b200 import _native as N
from paper_2605_29664_b200 import kernels as K


def med(fn, n=30, warm=5):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


T, h = 8192, 2048
CASES = [
    ("fc1_fwd", T, 4 * h, h, False, False, N.EPI_STORE_BF16),
    ("fc2_fwd", T, h, 4 * h, False, False, N.EPI_STORE_BF16),
    ("fc1_dgrad", T, h, 4 * h, False, True, N.EPI_STORE_BF16),
    ("fc1_dgrad_kmajor", T, h, 4 * h, False, False, N.EPI_STORE_BF16),
    ("fc1_wgrad", 4 * h, h, T, True, True, N.EPI_ACCUM_F32),
    ("fc1_wgrad_store", 4 * h, h, T, True, True, N.EPI_STORE_F32),
    ("fc1_wgrad_bf16", 4 * h, h, T, True, True, N.EPI_STORE_BF16),
    ("fc1_wgrad_kk", 4 * h, h, T, False, False, N.EPI_STORE_BF16),
    ("qkv_wgrad", 3 * h, h, T, True, True, N.EPI_ACCUM_F32),
    ("out_wgrad", h, h, T, True, True, N.EPI_ACCUM_F32),
    ("fc2_dgrad_gelubwd", T, 4 * h, h, False, True, N.EPI_GELU_BWD),
    ("fc1_wgrad_amn", 4 * h, h, T, True, False, N.EPI_STORE_BF16),
    ("fc1_wgrad_bmn", 4 * h, h, T, False, True, N.EPI_STORE_BF16),
    ("fc2_fwd_residual", T, h, 4 * h, False, False, N.EPI_RESIDUAL),
    ("fc1_fwd_gelu", T, 4 * h, h, False, False, N.EPI_GELU),
]
only = set(sys.argv[1:])
for name, M, Nn, Kk, a_mn, b_mn, epi in CASES:
    if only and name not in only:
        continue
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
    print(json.dumps(dict(kernel=name, ms=round(ms, 4), tflops=round(fl / ms / 1e9, 1),
                          torch_tflops=round(fl / ms_t / 1e9, 1))), flush=True)
