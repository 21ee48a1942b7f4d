"""fc1 weight gradient (8192 x 2048 x 8192) with MN-major operands (the executor's layout) and
with K-major operands, for an ncu comparison of the two load paths."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_29664_b200 import _native as N  # noqa: E402
from paper_2605_29664_b200 import kernels as K  # noqa: E402

T, h, F = 8192, 2048, 8192
dU = torch.randn(T, F, device="cuda").bfloat16()    # [T][F]
X = torch.randn(T, h, device="cuda").bfloat16()     # [T][h]
dUt = dU.T.contiguous()                              # [F][T]
Xt = X.T.contiguous()                                # [h][T]
C = torch.zeros(F, h, device="cuda")
for _ in range(2):
    K.gemm(dU, X, M=F, N_=h, K=T, a_mn=True, b_mn=True, C=C, epilogue=N.EPI_ACCUM_F32)    # MN, MN
    K.gemm(dUt, Xt, M=F, N_=h, K=T, a_mn=False, b_mn=False, C=C, epilogue=N.EPI_ACCUM_F32)  # K, K
torch.cuda.synchronize()
