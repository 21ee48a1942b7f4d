"""Times the stage kernels at the 1.3B (h=2048, T=8192) shapes with CUDA events.
Prints one line per kernel: shape, ms, TFLOP/s (or GB/s), and torch/cuBLAS for context."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_29664_b200 import kernels as K, _native as N

def timeit(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

T, h, V = 8192, 2048, 50304
res = []
def gemm_case(name, M, Nn, Kk, a_mn, b_mn, epi=N.EPI_STORE_BF16):
    A = torch.randn(Kk, M, device="cuda").bfloat16() if a_mn else torch.randn(M, Kk, device="cuda").bfloat16()
    B = torch.randn(Kk, Nn, device="cuda").bfloat16() if b_mn else torch.randn(Nn, Kk, device="cuda").bfloat16()
    dt = torch.float32 if epi == N.EPI_ACCUM_F32 else torch.bfloat16
    C = torch.zeros(M, Nn, dtype=dt, device="cuda")
    ms = timeit(lambda: K.gemm(A, B, M=M, N_=Nn, K=Kk, a_mn=a_mn, b_mn=b_mn, C=C, epilogue=epi))
    Al = A.T if a_mn else A
    Bl = B if b_mn else B.T
    ms_t = timeit(lambda: torch.matmul(Al, Bl))
    fl = 2.0 * M * Nn * Kk
    res.append(dict(kernel=name, shape=[M, Nn, Kk], ms=round(ms, 4), tflops=round(fl / ms / 1e9, 1),
                    torch_ms=round(ms_t, 4), torch_tflops=round(fl / ms_t / 1e9, 1)))
    print(json.dumps(res[-1]), flush=True)

gemm_case("qkv_fwd", T, 3 * h, h, False, False)
gemm_case("fc1_fwd_gelu", T, 4 * h, h, False, False)
gemm_case("fc2_fwd", T, h, 4 * h, False, False)
gemm_case("fc1_dgrad", T, h, 4 * h, False, True)
gemm_case("qkv_wgrad", 3 * h, h, T, True, True, N.EPI_ACCUM_F32)
gemm_case("fc1_wgrad", 4 * h, h, T, True, True, N.EPI_ACCUM_F32)
gemm_case("head_fwd", T, V, h, False, False)
gemm_case("square8192", 8192, 8192, 8192, False, False)

B, S, H, D = 4, 2048, 16, 128
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, S, H, D)
ms_f = timeit(lambda: K.attention_fwd(qkv, B, S, H, D))
ms_b = timeit(lambda: K.attention_bwd(qkv, out, dout, lse, B, S, H, D))
fl = 4.0 * B * H * S * S * D / 2  # causal
q, k, v = qkv.view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
ms_sdpa = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True))
print(json.dumps(dict(kernel="attn_fwd", ms=round(ms_f, 4), tflops=round(fl / ms_f / 1e9, 1), sdpa_ms=round(ms_sdpa, 4))))
print(json.dumps(dict(kernel="attn_bwd", ms=round(ms_b, 4), tflops=round(2.5 * fl / ms_b / 1e9, 1))))

x = torch.randn(T, h, device="cuda").bfloat16()
g = torch.ones(h, device="cuda"); b = torch.zeros(h, device="cuda")
ms = timeit(lambda: K.layernorm_fwd(x, g, b))
print(json.dumps(dict(kernel="ln_fwd", ms=round(ms, 4), gbs=round((4 * T * h + 8 * T) / ms / 1e6, 1))))
n = 151_000_000
th = torch.randn(n, device="cuda"); m = torch.zeros(n, device="cuda"); vv = torch.zeros(n, device="cuda")
gr = torch.randn(n, device="cuda"); w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
ms = timeit(lambda: K.optimizer_step(3, th, m, vv, gr, w, lr=1e-4), iters=5)
print(json.dumps(dict(kernel="adamw", ms=round(ms, 4), gbs=round(34 * n / ms / 1e6, 1))))
lg = torch.randn(T, V, device="cuda").bfloat16(); lab = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
ls = torch.zeros(1, device="cuda")
ms = timeit(lambda: K.xent_fwd_bwd(lg, lab, ls, 1.0), iters=5)
print(json.dumps(dict(kernel="xent", ms=round(ms, 4), gbs=round(3 * 2 * T * V / ms / 1e6, 1))))
