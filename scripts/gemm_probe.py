"""Runs the stage GEMMs of one 1.3B layer-minibatch (for ncu captures)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29664_b200 import kernels as K, _native as N
T, h = 8192, 2048
A = torch.randn(T, h, device="cuda").bfloat16(); W1 = torch.randn(4 * h, h, device="cuda").bfloat16()
G = torch.randn(T, 4 * h, device="cuda").bfloat16(); X = torch.randn(T, h, device="cuda").bfloat16()
Cf = torch.zeros(4 * h, h, device="cuda")
for _ in range(3):
    K.gemm(A, W1, M=T, N_=4 * h, K=h)                                    # fc1-shaped forward
    K.gemm(G, X, M=4 * h, N_=h, K=T, a_mn=True, b_mn=True, C=Cf, epilogue=N.EPI_ACCUM_F32)  # fc1 wgrad
torch.cuda.synchronize()
