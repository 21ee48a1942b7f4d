"""Sustained (power-capped) GEMM throughput: each case runs back to back for ~3 s while
nvidia-smi samples SM clock and power; prints TFLOP/s, median clock and median power, for
amdp_gemm and for torch.matmul (cuBLAS) on the same logical product.  Under the 1 kW cap
the sustained rate is energy-bound, so TFLOP/s per watt is the figure of merit."""
import json
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_29664_b200 import _native as N
from paper_2605_29664_b200 import kernels as K

T, h = 8192, 2048
CASES = {
    "fc1_fwd": (T, 4 * h, h, False, False, N.EPI_STORE_BF16),
    "fc1_dgrad": (T, h, 4 * h, False, True, N.EPI_STORE_BF16),
    "fc1_wgrad": (4 * h, h, T, True, True, N.EPI_ACCUM_F32),
    "square8192": (8192, 8192, 8192, False, False, N.EPI_STORE_BF16),
    "fc1_dgrad_kk": (T, h, 4 * h, False, False, N.EPI_STORE_BF16),
    "fc1_wgrad_kk": (4 * h, h, T, False, False, N.EPI_STORE_BF16),
    "fc1_wgrad_bf16": (4 * h, h, T, True, True, N.EPI_STORE_BF16),
    "fc2_fwd": (T, h, 4 * h, False, False, N.EPI_STORE_BF16),
    "fc1_wgrad_amn": (4 * h, h, T, True, False, N.EPI_ACCUM_F32),
    "fc1_fwd_amn": (T, 4 * h, h, True, False, N.EPI_STORE_BF16),
    "fc2_fwd_amn": (T, h, 4 * h, True, False, N.EPI_STORE_BF16),
}


def sustained(fn, flops, secs=3.0):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "-i", str(torch.cuda.current_device()),
                            "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.PIPE, text=True)
    n = 0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.time()
    s.record()
    while time.time() - t0 < secs:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    smi.terminate()
    out, _ = smi.communicate()
    rows = [list(map(float, l.split(","))) for l in out.strip().splitlines() if l.strip()]
    rows = rows[len(rows) // 4:]  # settled part
    ms = s.elapsed_time(e) / n
    return dict(tflops=round(flops / ms / 1e9, 1), sm_mhz=statistics.median(r[0] for r in rows),
                watts=statistics.median(r[1] for r in rows))


only = set(sys.argv[1:])
for name, (M, Nn, Kk, a_mn, b_mn, epi) in CASES.items():
    if only and name not in only:
        continue
    A = torch.randn(Kk, M, device="cuda").bfloat16() if a_mn else torch.randn(M, Kk, device="cuda").bfloat16()
    B = torch.randn(Kk, Nn, device="cuda").bfloat16() if b_mn else torch.randn(Nn, Kk, device="cuda").bfloat16()
    dt = torch.float32 if epi == N.EPI_ACCUM_F32 else torch.bfloat16
    C = torch.zeros(M, Nn, dtype=dt, device="cuda")
    fl = 2.0 * M * Nn * Kk
    ours = sustained(lambda: K.gemm(A, B, M=M, N_=Nn, K=Kk, a_mn=a_mn, b_mn=b_mn, C=C, epilogue=epi), fl)
    Al = A.T if a_mn else A
    Bl = B if b_mn else B.T
    cub = sustained(lambda: torch.matmul(Al, Bl), fl)
    print(json.dumps({"case": name, "ours": ours, "cublas": cub}), flush=True)
