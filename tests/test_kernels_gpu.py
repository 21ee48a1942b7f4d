"""GPU parity of every sm_100a kernel against a plain PyTorch fp32 restatement of the same op.

Tolerances are stated per test: bf16 outputs carry ~2^-8 relative rounding, fp32
accumulation order differs from torch's.
"""
import ctypes
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2605_29664_b200 import kernels
    return kernels


@pytest.fixture(scope="module")
def N():
    from paper_2605_29664_b200 import _native
    return _native


def _rel(a, b):
    a = a.double()
    b = b.double()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


GEMM_SHAPES = [(256, 384, 128), (1000, 520, 192), (4096, 3072, 1024), (384, 50304, 256)]


@pytest.mark.parametrize("M,N_,K_", GEMM_SHAPES)
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_store(K, N, M, N_, K_, a_mn, b_mn):
    torch.manual_seed(0)
    A = torch.randn(M, K_, device="cuda").bfloat16()
    B = torch.randn(N_, K_, device="cuda").bfloat16()
    ref = A.float() @ B.float().T
    As = A.T.contiguous() if a_mn else A
    Bs = B.T.contiguous() if b_mn else B
    C = K.gemm(As, Bs, M=M, N_=N_, K=K_, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    assert _rel(C, ref) < 8e-3


# Shapes whose last wave is split along N (tail_split 2 or 4 over 74 CTA pairs):
# 8192x2048 = 256 tiles (R=34 -> s=2); 2560x2000 = 80 tiles (R=6 -> s=4 for K-major B,
# partial last N tile); 6144x2048 = 192 tiles (R=44 -> s=4 K-major).  Every element is
# checked, so a missing or misplaced sub-tile fails.
@pytest.mark.parametrize("M,N_,K_", [(8192, 2048, 128), (2560, 2000, 128), (6144, 2048, 192)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("accum", [False, True])
def test_gemm_split_tail(K, N, M, N_, K_, a_mn, b_mn, accum):
    torch.manual_seed(3)
    A = torch.randn(M, K_, device="cuda").bfloat16()
    B = torch.randn(N_, K_, device="cuda").bfloat16()
    ref = A.float() @ B.float().T
    As = A.T.contiguous() if a_mn else A
    Bs = B.T.contiguous() if b_mn else B
    if accum:
        C0 = torch.randn(M, N_, device="cuda")
        C = C0.clone()
        K.gemm(As, Bs, M=M, N_=N_, K=K_, a_mn=a_mn, b_mn=b_mn, C=C, epilogue=N.EPI_ACCUM_F32)
        ref = ref + C0
        tol = 1e-3
    else:
        C = K.gemm(As, Bs, M=M, N_=N_, K=K_, a_mn=a_mn, b_mn=b_mn)
        tol = 0.02 * ref.abs().max().item()
    torch.cuda.synchronize()
    err = (C.float() - ref).abs().max().item()
    assert err < tol, f"max abs err {err}"


# Weight-gradient shape with a partial last wave that fits in one wave as K halves (fc1 at
# 1.3B: 256 tiles on 74 pairs -> 34 tail tiles split in two; LM-head-like 1576 tiles): every
# element checked, and the fp32 result is bitwise reproducible (the second K half adds after
# the first, in a fixed order).
@pytest.mark.parametrize("M,N_,K_", [(8192, 2048, 1024), (2048, 50304, 512)])
def test_gemm_accum_ksplit_tail_deterministic(K, N, M, N_, K_):
    torch.manual_seed(9)
    A = torch.randn(K_, M, device="cuda").bfloat16()   # MN-major (activation gradient^T)
    B = torch.randn(K_, N_, device="cuda").bfloat16()  # MN-major (activations)
    C0 = torch.randn(M, N_, device="cuda")
    ref = C0.double() + (A.double().T @ B.double())
    outs = []
    for _ in range(3):
        C = C0.clone()
        K.gemm(A, B, M=M, N_=N_, K=K_, a_mn=True, b_mn=True, C=C, epilogue=N.EPI_ACCUM_F32)
        torch.cuda.synchronize()
        outs.append(C)
    err = (outs[0].double() - ref).abs().max().item()
    assert err < 1e-3 * ref.abs().max().item(), err
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


# Small products on single-CTA tiles (BERT-large shapes, < 20 GFLOP): 128 x 256 by default,
# 128 x 128 under AMDP_GEMM_NARROW (test_gemm_narrow_tiles_subprocess):
# BERT-large shapes (fc2 forward: 64 tiles of 128 x 256 -> 128 tiles of 128 x 128; the
# out-projection weight gradient, MN-major operands) and a ragged one (partial M and N tiles),
# every epilogue, every element checked against torch fp32, and bitwise reproducible.
SMALL_SHAPES = [(2048, 1024, 4096, False, False), (1024, 1024, 2048, True, True), (1000, 776, 1472, False, True)]


@pytest.mark.parametrize("M,N_,K_,a_mn,b_mn", SMALL_SHAPES)
@pytest.mark.parametrize("epi", ["store", "gelu", "residual", "gelu_bwd", "accum", "store_f32"])
def test_gemm_small_tiles(K, N, M, N_, K_, a_mn, b_mn, epi):
    torch.manual_seed(11)
    A = torch.randn(M, K_, device="cuda").bfloat16()
    B = (torch.randn(N_, K_, device="cuda") / math.sqrt(K_)).bfloat16()
    As = A.T.contiguous() if a_mn else A
    Bs = B.T.contiguous() if b_mn else B
    prod = A.float() @ B.float().T
    aux = torch.randn(M, N_, device="cuda").bfloat16()
    outs = []
    for _ in range(2):
        kw = {}
        if epi == "store":
            kw = dict(epilogue=N.EPI_STORE_BF16)
        elif epi == "gelu":
            kw = dict(epilogue=N.EPI_GELU, C2=torch.empty(M, N_, dtype=torch.bfloat16, device="cuda"), ldc2=N_)
        elif epi == "residual":
            kw = dict(epilogue=N.EPI_RESIDUAL, aux=aux, ld_aux=N_)
        elif epi == "gelu_bwd":
            kw = dict(epilogue=N.EPI_GELU_BWD, aux=aux, ld_aux=N_)
        elif epi == "accum":
            kw = dict(epilogue=N.EPI_ACCUM_F32, C=torch.ones(M, N_, device="cuda"))
        else:
            kw = dict(epilogue=N.EPI_STORE_F32)
        C = K.gemm(As, Bs, M=M, N_=N_, K=K_, a_mn=a_mn, b_mn=b_mn, **kw)
        torch.cuda.synchronize()
        outs.append((C.clone(), kw.get("C2")))
    C, C2 = outs[0]
    if epi == "gelu":
        ref, ref2 = _gelu(C2.float()), prod
        assert (C2.float() - ref2).abs().max().item() < 0.02 * ref2.abs().max().item()
    elif epi == "residual":
        ref = prod + aux.float()
    elif epi == "gelu_bwd":
        x = aux.float()
        t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
        ref = prod * (0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x))
    elif epi == "accum":
        ref = prod + 1.0
    else:
        ref = prod
    tol = (1e-4 if epi in ("accum", "store_f32") else 0.02) * ref.abs().max().item()
    err = (C.float() - ref).abs().max().item()
    assert err < tol, f"max abs err {err} (tol {tol})"
    assert torch.equal(outs[0][0], outs[1][0])


def test_gemm_narrow_tiles_subprocess():
    """AMDP_GEMM_NARROW=2 (128 x 128 single-CTA tiles everywhere below the pair threshold) is
    read once per process: the small-tile and rowdot cases re-run in a child process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AMDP_GEMM_NARROW="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_kernels_gpu.py"), "-k", "small_tiles or rowdot or gemm_store"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (True, True)])
def test_gemm_accum_f32(K, N, a_mn, b_mn):
    torch.manual_seed(1)
    M, N_, K_ = 768, 1024, 512
    A = torch.randn(M, K_, device="cuda").bfloat16()
    B = torch.randn(N_, K_, device="cuda").bfloat16()
    C0 = torch.randn(M, N_, device="cuda")
    ref = C0 + 0.5 * (A.float() @ B.float().T)
    As = A.T.contiguous() if a_mn else A
    Bs = B.T.contiguous() if b_mn else B
    C = C0.clone()
    K.gemm(As, Bs, M=M, N_=N_, K=K_, a_mn=a_mn, b_mn=b_mn, C=C, epilogue=N.EPI_ACCUM_F32,
           alpha=0.5)
    torch.cuda.synchronize()
    assert _rel(C, ref) < 1e-5


def _gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def test_gemm_gelu_residual_gelubwd(K, N):
    torch.manual_seed(2)
    M, N_, K_ = 512, 768, 256
    A = (0.1 * torch.randn(M, K_, device="cuda")).bfloat16()
    B = torch.randn(N_, K_, device="cuda").bfloat16()
    acc = A.float() @ B.float().T
    pre = torch.empty(M, N_, dtype=torch.bfloat16, device="cuda")
    C = K.gemm(A, B, M=M, N_=N_, K=K_, epilogue=N.EPI_GELU, C2=pre, ldc2=N_)
    torch.cuda.synchronize()
    assert _rel(pre, acc) < 8e-3
    assert _rel(C, _gelu(acc)) < 1e-2
    R = torch.randn(M, N_, device="cuda").bfloat16()
    C = K.gemm(A, B, M=M, N_=N_, K=K_, epilogue=N.EPI_RESIDUAL, aux=R, ld_aux=N_)
    torch.cuda.synchronize()
    assert _rel(C, acc + R.float()) < 8e-3
    U = torch.randn(M, N_, device="cuda").bfloat16()
    x = U.float().requires_grad_()
    _gelu(x).backward(acc)
    C = K.gemm(A, B, M=M, N_=N_, K=K_, epilogue=N.EPI_GELU_BWD, aux=U, ld_aux=N_)
    torch.cuda.synchronize()
    assert _rel(C, x.grad) < 1e-2


@pytest.mark.parametrize("shape", [(512, 768, 256), (2048, 2048, 1024)])
def test_recompute_gelu_bit_identical_to_epilogue(K, N, shape):
    """The recompute path's f = gelu(u) (amdp_gelu_fwd on the stored bf16 pre-activation) is
    bit-identical to the fc1 GEMM epilogue's f: both take gelu of the bf16-rounded u with the
    same spelled-out operations, so recomputation changes no bit of the backward's inputs."""
    torch.manual_seed(3)
    M, N_, K_ = shape
    A = (0.05 * torch.randn(M, K_, device="cuda")).bfloat16()
    B = torch.randn(N_, K_, device="cuda").bfloat16()
    u = torch.empty(M, N_, dtype=torch.bfloat16, device="cuda")
    f_epi = K.gemm(A, B, M=M, N_=N_, K=K_, epilogue=N.EPI_GELU, C2=u, ldc2=N_)
    f_re = torch.empty_like(f_epi)
    N.check(N.lib.amdp_gelu_fwd(ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f_re.data_ptr()),
                                ctypes.c_int64(M * N_), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
            "amdp_gelu_fwd")
    torch.cuda.synchronize()
    assert torch.equal(f_epi.view(torch.int16), f_re.view(torch.int16))
    assert _rel(f_re, _gelu(u.float())) < 1e-2


def _attn_ref(qkv, B, S, H, D, causal, key_len=None):
    q, k, v = qkv.float().view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    s = q @ k.transpose(-1, -2) / math.sqrt(D)
    if causal:
        mask = torch.ones(S, S, dtype=torch.bool, device=qkv.device).triu(1)
        s = s.masked_fill(mask, float("-inf"))
    if key_len is not None:  # [B] valid key count per sequence
        kpad = torch.arange(S, device=qkv.device)[None, :] >= key_len[:, None].long()
        s = s.masked_fill(kpad[:, None, None, :], float("-inf"))
    p = s.softmax(-1)
    o = p @ v  # B H S D
    return o.permute(0, 2, 1, 3).reshape(B * S, H * D)


@pytest.mark.parametrize("B,S,H,D", [(2, 128, 4, 32), (4, 64, 4, 32), (3, 64, 2, 64), (2, 128, 3, 64), (2, 256, 3, 64),
                                     (2, 512, 3, 80), (1, 2048, 2, 80), (2, 256, 2, 128), (4, 2048, 2, 128)])
@pytest.mark.parametrize("causal", [True, False])
def test_attention_fwd_bwd(K, B, S, H, D, causal):
    torch.manual_seed(3)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, S, H, D, causal)
    x = qkv.float().requires_grad_()
    ref = _attn_ref(x, B, S, H, D, causal)
    ref.backward(dout.float())
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-2
    dqkv = K.attention_bwd(qkv, out, dout, lse, B, S, H, D, causal)
    torch.cuda.synchronize()
    g = x.grad
    hd = H * D
    for part in range(3):
        assert _rel(dqkv[:, part * hd:(part + 1) * hd], g[:, part * hd:(part + 1) * hd]) < 2e-2


@pytest.mark.parametrize("B,S,H,D", [(3, 128, 4, 32), (3, 64, 4, 32), (3, 128, 2, 64), (3, 256, 3, 64), (3, 512, 2, 128),
                                     (2, 512, 2, 80)])
def test_attention_key_padding(K, B, S, H, D):
    """Bidirectional attention with key_len[b] (BERT padding): keys >= key_len[b] get zero
    probability; their dK / dV are exactly zero.  Lengths cover a full tile, a ragged tail
    inside the first tile and a single valid key."""
    torch.manual_seed(8)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    lens = [S, S // 2 + 17, 1, 100][:B]
    key_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out, lse = K.attention_fwd(qkv, B, S, H, D, False, key_len=key_len)
    x = qkv.float().requires_grad_()
    ref = _attn_ref(x, B, S, H, D, False, key_len)
    ref.backward(dout.float())
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-2
    dqkv = K.attention_bwd(qkv, out, dout, lse, B, S, H, D, False, key_len=key_len)
    torch.cuda.synchronize()
    hd = H * D
    for part in range(3):
        assert _rel(dqkv[:, part * hd:(part + 1) * hd], x.grad[:, part * hd:(part + 1) * hd]) < 2e-2
    for b, n in enumerate(lens):  # padded keys: dK = dV = 0 exactly
        assert not dqkv[b * S + n:(b + 1) * S, hd:].any()
    with pytest.raises(RuntimeError):  # causal + key padding is not a supported combination
        K.attention_fwd(qkv, B, S, H, D, True, key_len=key_len)


def test_attention_impl_report(K, N):
    """Every BASELINE model shape (and the tiny configuration) runs a tcgen05 kernel; shapes
    neither the tiled nor the one-tile kernels take are rejected (no fallback path)."""
    T = N.ATTN_IMPL_TCGEN05
    for S, D in [(64, 32), (128, 32), (64, 64), (128, 64), (512, 64), (1024, 64), (2048, 128), (2048, 80)]:
        assert N.lib.amdp_attention_impl(S, D, 0) == T and N.lib.amdp_attention_impl(S, D, 1) == T, (S, D)
    assert N.lib.amdp_attention_impl(192, 80, 0) == -1 and N.lib.amdp_attention_impl(128, 128, 0) == -1
    qkv = torch.randn(192, 3 * 2 * 80, device="cuda").bfloat16()
    with pytest.raises(RuntimeError):
        K.attention_fwd(qkv, 1, 192, 2, 80, True)


# (M, N, K, seg, seq): the 1.3B dO GEMM (8192x2048, 256 tiles -> tail split), a 350M-like
# head_dim 64 case, a single-CTA M < 256 case and a 64-wide-tail case (segments split
# between two CTAs: atomic sum of two partials onto zero).
@pytest.mark.parametrize("M,N_,K_,seg,seq", [(8192, 2048, 256, 128, 2048), (4096, 1024, 128, 64, 1024),
                                             (128, 512, 128, 128, 64), (2560, 2048, 128, 128, 512),
                                             (2048, 1024, 1024, 64, 512)])  # BERT-large dO: 128 x 128 tiles
def test_gemm_rowdot(K, N, M, N_, K_, seg, seq):
    """AMDP_EPI_ROWDOT: C = bf16(A B^T) and rowdot[b][h][s] = sum over the h-th seg-column
    segment of bf16(C) * aux (attention backward's delta from the dO GEMM)."""
    torch.manual_seed(5)
    A = torch.randn(M, K_, device="cuda").bfloat16()
    B = (torch.randn(N_, K_, device="cuda") / math.sqrt(K_)).bfloat16()
    aux = torch.randn(M, N_, device="cuda").bfloat16()
    rowdot = torch.full((M // seq, N_ // seg, seq), float("nan"), device="cuda")
    C = K.gemm(A, B, M=M, N_=N_, K=K_, epilogue=N.EPI_ROWDOT, aux=aux, ld_aux=N_, rowdot=rowdot,
               rowdot_seg=seg, rowdot_seq=seq)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    assert (C.float() - ref).abs().max().item() < 0.02 * ref.abs().max().item()
    want = (C.float() * aux.float()).view(M // seq, seq, N_ // seg, seg).sum(-1).permute(0, 2, 1)
    assert torch.isfinite(rowdot).all()
    assert _rel(rowdot, want) < 1e-5


@pytest.mark.parametrize("B,S,H,D", [(2, 256, 3, 64), (4, 2048, 2, 128), (1, 512, 2, 80), (4, 64, 4, 32), (2, 64, 3, 64)])
@pytest.mark.parametrize("causal", [True, False])
def test_attention_bwd_supplied_delta(K, B, S, H, D, causal):
    """amdp_attention_bwd_delta with delta = rowsum(dO * O) from the caller gives the same
    gradients as the self-contained backward (torch fp32 reference as above)."""
    torch.manual_seed(6)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    out, lse = K.attention_fwd(qkv, B, S, H, D, causal)
    delta = (dout.float() * out.float()).view(B, S, H, D).sum(-1).permute(0, 2, 1).contiguous()
    dqkv = K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, causal)
    x = qkv.float().requires_grad_()
    _attn_ref(x, B, S, H, D, causal).backward(dout.float())
    torch.cuda.synchronize()
    hd = H * D
    for part in range(3):
        assert _rel(dqkv[:, part * hd:(part + 1) * hd], x.grad[:, part * hd:(part + 1) * hd]) < 2e-2


@pytest.mark.parametrize("B,S,H,D,causal,padded", [(2, 256, 3, 64, True, False), (4, 2048, 2, 128, True, False),
                                                    (1, 512, 2, 80, True, False), (2, 768, 2, 128, False, False),
                                                    (4, 512, 3, 64, False, True), (3, 1024, 2, 64, True, False),
                                                    (1, 256, 2, 128, True, False), (2, 2048, 2, 80, False, False)])
def test_attention_bwd_ds_scratch(K, N, B, S, H, D, causal, padded):
    """The engine's backward (dK/dV kernel stores dS^T chunks, dQ = dS K by fa_bwd_dq_gemm_kernel)
    against torch fp32 and against the dQ kernel that recomputes S / dP: dK and dV come from the
    same kernel (bit-identical), dQ agrees within bf16 rounding, and two runs are bit-identical
    (no atomics).  Covers head_dim 64 / 80 / 128, causal and bidirectional, a single query tile,
    a non-power-of-two tile count and BERT key padding."""
    torch.manual_seed(11)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    key_len = torch.tensor([S, S // 2 + 17, 1, 100][:B], dtype=torch.int32, device="cuda") if padded else None
    out, lse = K.attention_fwd(qkv, B, S, H, D, causal, key_len=key_len)
    delta = (dout.float() * out.float()).view(B, S, H, D).sum(-1).permute(0, 2, 1).contiguous()
    assert N.lib.amdp_attention_bwd_scratch_bytes(B, S, H, D, int(causal)) == (0 if D == 80 else B * H * 16384 * (
        (S // 128) * (S // 128 + 1) if causal else 2 * (S // 128) ** 2))
    d1 = K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, causal, key_len=key_len)
    d2 = K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, causal, key_len=key_len)
    d0 = K.attention_bwd_delta(qkv, dout, lse, delta, B, S, H, D, causal, key_len=key_len, scratch=False)
    x = qkv.float().requires_grad_()
    _attn_ref(x, B, S, H, D, causal, key_len).backward(dout.float())
    torch.cuda.synchronize()
    hd = H * D
    assert torch.equal(d1, d2)
    assert torch.equal(d1[:, hd:], d0[:, hd:])
    assert _rel(d1[:, :hd], d0[:, :hd]) < 5e-3
    for part in range(3):
        assert _rel(d1[:, part * hd:(part + 1) * hd], x.grad[:, part * hd:(part + 1) * hd]) < 2e-2


@pytest.mark.parametrize("rows,cols", [(256, 128), (1000, 1024), (4096, 2048), (512, 2560)])
def test_layernorm(K, rows, cols):
    torch.manual_seed(4)
    x = (torch.randn(rows, cols, device="cuda") * 2 + 0.5).bfloat16()
    gamma = 1 + 0.1 * torch.randn(cols, device="cuda")
    beta = 0.1 * torch.randn(cols, device="cuda")
    y, mean, rstd = K.layernorm_fwd(x, gamma, beta)
    xf = x.float().requires_grad_()
    g = gamma.clone().requires_grad_()
    b = beta.clone().requires_grad_()
    ref = torch.nn.functional.layer_norm(xf, (cols,), g, b, 1e-5)
    dy = torch.randn(rows, cols, device="cuda").bfloat16()
    ref.backward(dy.float())
    torch.cuda.synchronize()
    assert _rel(y, ref) < 8e-3
    resid = torch.randn(rows, cols, device="cuda").bfloat16()
    dg = torch.ones(cols, device="cuda")
    db = torch.zeros(cols, device="cuda")
    dx = K.layernorm_bwd(dy, x, gamma, mean, rstd, resid, dg, db)
    torch.cuda.synchronize()
    assert _rel(dx, xf.grad + resid.float()) < 1e-2
    assert _rel(dg - 1, g.grad) < 1e-3
    assert _rel(db, b.grad) < 1e-3


@pytest.mark.parametrize("rows,cols", [(2048, 1024), (8192, 2048), (1000, 512)])
def test_layernorm_deferred_param_grads(K, rows, cols):
    """amdp_layernorm_bwd_rows over 3 calls (a window of minibatches) + one flush: dx equals
    amdp_layernorm_bwd's bit for bit, dgamma / dbeta equal the per-call reductions' sum
    within fp32 reassociation (and torch's), the partial rows are zero again after the
    flush, and the whole sequence is bitwise reproducible."""
    torch.manual_seed(12)
    parts = K.layernorm_bwd_parts(rows, cols)
    assert parts > 0
    gamma = 1 + 0.1 * torch.randn(cols, device="cuda")
    beta = 0.1 * torch.randn(cols, device="cuda")
    xs = [(torch.randn(rows, cols, device="cuda") * 2 + 0.5).bfloat16() for _ in range(3)]
    dys = [torch.randn(rows, cols, device="cuda").bfloat16() for _ in range(3)]
    resid = torch.randn(rows, cols, device="cuda").bfloat16()
    stats = [K.layernorm_fwd(x, gamma, beta)[1:] for x in xs]

    def deferred():
        part = torch.zeros(parts, 2, cols, device="cuda")
        dg = torch.full((cols,), 0.5, device="cuda")
        db = torch.zeros(cols, device="cuda")
        dxs = [K.layernorm_bwd_rows(dy, x, gamma, m, r, resid, part) for dy, x, (m, r) in zip(dys, xs, stats)]
        K.layernorm_dgb_flush(part, parts, cols, dg, db)
        torch.cuda.synchronize()
        assert not part.any()
        return dxs, dg, db

    dxs, dg, db = deferred()
    dg0 = torch.full((cols,), 0.5, device="cuda")
    db0 = torch.zeros(cols, device="cuda")
    for i, (dy, x, (m, r)) in enumerate(zip(dys, xs, stats)):
        dx0 = K.layernorm_bwd(dy, x, gamma, m, r, resid, dg0, db0)
        torch.cuda.synchronize()
        assert torch.equal(dx0, dxs[i])
    assert _rel(dg - 0.5, dg0 - 0.5) < 1e-5 and _rel(db, db0) < 1e-5
    dg_ref = sum(((x.float() - m[:, None]) * r[:, None] * dy.float()).sum(0) for dy, x, (m, r) in zip(dys, xs, stats))
    assert _rel(dg - 0.5, dg_ref) < 1e-4
    dxs2, dg2, db2 = deferred()
    assert torch.equal(dg, dg2) and torch.equal(db, db2)


def test_embedding(K):
    torch.manual_seed(5)
    V, S, Bn, Hd = 1000, 64, 4, 256
    wte = torch.randn(V, Hd, device="cuda").bfloat16()
    wpe = torch.randn(S, Hd, device="cuda").bfloat16()
    tok = torch.randint(0, V, (Bn * S,), device="cuda", dtype=torch.int32)
    x = K.embedding_fwd(tok, wte, wpe, S)
    pos = torch.arange(Bn * S, device="cuda") % S
    ref = wte.float()[tok.long()] + wpe.float()[pos]
    torch.cuda.synchronize()
    assert _rel(x, ref) < 4e-3
    dx = torch.randn(Bn * S, Hd, device="cuda").bfloat16()
    dwte = torch.zeros(V, Hd, device="cuda")
    dwpe = torch.zeros(S, Hd, device="cuda")
    K.embedding_bwd(tok, dx, dwte, dwpe, S)
    rte = torch.zeros(V, Hd, device="cuda").index_add_(0, tok.long(), dx.float())
    rpe = dx.float().view(Bn, S, Hd).sum(0)
    torch.cuda.synchronize()
    assert _rel(dwte, rte) < 1e-5
    assert _rel(dwpe, rpe) < 1e-5


@pytest.mark.parametrize("ntok,S,V,Hd", [(2048, 512, 30528, 1024), (8192, 2048, 50304, 256), (16384, 2048, 50304, 64)])
def test_embedding_bwd_deterministic(K, ntok, S, V, Hd):
    """The token-table gradient has no atomics: heavily repeated tokens (a BERT [MASK]-like id on
    15% of positions) give bitwise-identical results run to run and match the fp32 sum; the
    largest supported minibatch (16384 tokens) works."""
    torch.manual_seed(8)
    tok = torch.randint(0, V, (ntok,), device="cuda", dtype=torch.int32)
    tok[torch.rand(ntok, device="cuda") < 0.15] = V - 1
    dx = torch.randn(ntok, Hd, device="cuda").bfloat16()
    outs = []
    for _ in range(3):
        dwte = torch.full((V, Hd), 0.25, device="cuda")
        dwpe = torch.zeros(S, Hd, device="cuda")
        K.embedding_bwd(tok, dx, dwte, dwpe, S)
        outs.append(dwte)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    rte = torch.full((V, Hd), 0.25, device="cuda", dtype=torch.float64).index_add_(0, tok.long(), dx.double())
    assert _rel(outs[0], rte) < 1e-6


def test_embedding_bwd_sequential_order(K):
    """Each token's rows are summed in position order starting from zero, then added to the
    table: bit-identical to that sequential fp32 sum (numpy), also for a run of several hundred
    rows (a BERT padding-token run; the kernel batches its row loads) and runs of every length
    around the 8-row batching boundary."""
    import numpy as np
    torch.manual_seed(10)
    ntok, S, V, Hd = 2048, 512, 64, 64
    tok = torch.randint(1, V, (ntok,), device="cuda", dtype=torch.int32)
    tok[torch.rand(ntok, device="cuda") < 0.3] = 0  # one long run
    for n in range(1, 18):  # tokens 40 + n: runs of exactly n rows
        tok[(n * 97) % 1500:(n * 97) % 1500 + n] = 40 + n
    dx = torch.randn(ntok, Hd, device="cuda").bfloat16()
    dwte = torch.full((V, Hd), 0.25, device="cuda")
    dwpe = torch.zeros(S, Hd, device="cuda")
    K.embedding_bwd(tok, dx, dwte, dwpe, S)
    torch.cuda.synchronize()
    t = tok.cpu().numpy()
    x = dx.float().cpu().numpy()
    acc = np.zeros((V, Hd), dtype=np.float32)
    for p in range(ntok):  # position order within every token's run
        acc[t[p]] += x[p]
    want = np.float32(0.25) + acc
    assert np.array_equal(dwte.cpu().numpy(), want)


def test_xent_loss_deterministic(K):
    """The loss sum is a fixed-order reduction of per-row losses: bitwise repeatable."""
    torch.manual_seed(9)
    ntok, V = 4096, 50304
    logits = (3 * torch.randn(ntok, V, device="cuda")).bfloat16()
    labels = torch.randint(0, V, (ntok,), device="cuda", dtype=torch.int32)
    vals = []
    for _ in range(3):
        loss = torch.zeros(1, device="cuda")
        K.xent_fwd_bwd(logits.clone(), labels, loss, 1.0 / ntok)
        vals.append(loss.item())
    assert vals[0] == vals[1] == vals[2]


@pytest.mark.parametrize("ntok,V", [(256, 1024), (512, 50304), (64, 30528)])
def test_xent(K, ntok, V):
    torch.manual_seed(6)
    logits = (3 * torch.randn(ntok, V, device="cuda")).bfloat16()
    labels = torch.randint(0, V, (ntok,), device="cuda", dtype=torch.int32)
    labels[::7] = -1
    lf = logits.float().requires_grad_()
    valid = labels >= 0
    ref = torch.nn.functional.cross_entropy(lf[valid], labels[valid].long(), reduction="sum")
    scale = 1.0 / ntok
    (ref * scale).backward()
    loss = torch.zeros(1, device="cuda")
    lg = logits.clone()
    K.xent_fwd_bwd(lg, labels, loss, scale)
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) / ref.item() < 1e-4
    assert _rel(lg, lf.grad) < 1e-2


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_optimizer(K, N, kind):
    torch.manual_seed(7)
    n = 100003
    th = torch.randn(n, device="cuda")
    m = 0.01 * torch.randn(n, device="cuda")
    v = 0.01 * torch.rand(n, device="cuda")
    g = torch.randn(n, device="cuda")
    w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    T, M_, V_, G = th.double(), m.double(), v.double(), g.double() * 0.5
    lr, b1, b2, eps, wd = 0.01, 0.9, 0.999, 1e-3, 0.1
    if kind == 0:
        T = T - lr * G
    elif kind == 1:
        M_ = b1 * M_ + (1 - b1) * G
        T = T - lr * M_
    elif kind == 2:
        M_ = b1 * M_ + (1 - b1) * G
        V_ = b2 * V_ + (1 - b2) * G * G
        P = (1 / (V_.sqrt() + eps)).clamp(1e-8, 1e6)
        T = T - lr * P * M_
    else:
        step = 3
        M_ = b1 * M_ + (1 - b1) * G
        V_ = b2 * V_ + (1 - b2) * G * G
        mh, vh = M_ / (1 - b1 ** step), V_ / (1 - b2 ** step)
        T = T - lr * (mh / (vh.sqrt() + eps) + wd * T)
    K.optimizer_step(kind, th, m, v, g, w, lr=lr, beta1=b1, beta2=b2, eps=eps,
                     weight_decay=wd if kind == 3 else 0.0, grad_scale=0.5, step=3)
    torch.cuda.synchronize()
    assert torch.allclose(th.double(), T, rtol=1e-5, atol=1e-6)
    assert torch.equal(w, th.bfloat16())
    assert torch.count_nonzero(g).item() == 0


def _optim_gold():
    import json, os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "optim_golden.json")))


@pytest.mark.parametrize("case", _optim_gold(), ids=lambda c: c["name"])
def test_optimizer_kernel_vs_reference_apply_update(K, N, case):
    """amdp_optimizer_step (fp32) against ppsim::detail::apply_update (fp64, the reference's
    own code, optim.hpp:234-268) on the committed golden vectors; tolerance 2e-6 relative
    to the parameter scale (fp32 state, 5 steps)."""
    kind = {"sgd": 0, "momentum": 1}.get(case["name"], 2)
    th = torch.tensor(case["theta0"], dtype=torch.float32, device="cuda")
    m = torch.zeros_like(th)
    v = torch.zeros_like(th)
    w = torch.empty(th.numel(), dtype=torch.bfloat16, device="cuda")
    for g, want in zip(case["grads"], case["iterates"]):
        gr = torch.tensor(g, dtype=torch.float32, device="cuda")
        K.optimizer_step(kind, th, m, v, gr, w, lr=case["eta"], beta1=case["beta1"], beta2=case["beta2"],
                         eps=case["epsilon"], clamp_min=case["clamp_min"], clamp_max=case["clamp_max"])
        torch.cuda.synchronize()
        ref = torch.tensor(want, dtype=torch.float64, device="cuda")
        assert ((th.double() - ref).abs().max() / ref.abs().max()).item() < 2e-6
