"""Torch-tensor conveniences over the kernel C-ABI (include/amdp_kernels.h).

Torch is used only for device memory and the current stream; every call goes through
libamdp.so.  These wrappers are what the GPU parity tests call.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native as N


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def gemm(A, B, *, M, N_, K, a_mn=False, b_mn=False, lda=None, ldb=None, C=None, ldc=None,
         epilogue=N.EPI_STORE_BF16, aux=None, ld_aux=0, C2=None, ldc2=0, alpha=1.0,
         rowdot=None, rowdot_seg=0, rowdot_seq=0):
    """C = epi(alpha * A(m,k) B(n,k)); see amdp_gemm for the operand conventions."""
    if lda is None:
        lda = M if a_mn else K
    if ldb is None:
        ldb = N_ if b_mn else K
    if C is None:
        dt = torch.float32 if epilogue in (N.EPI_ACCUM_F32, N.EPI_STORE_F32) else torch.bfloat16
        C = torch.zeros(M, N_, dtype=dt, device=A.device)
    if ldc is None:
        ldc = C.stride(0)
    args = N.GemmArgs(M, N_, K, A.data_ptr(), lda, int(a_mn), B.data_ptr(), ldb, int(b_mn),
                      C.data_ptr(), ldc, aux.data_ptr() if aux is not None else 0, ld_aux,
                      C2.data_ptr() if C2 is not None else 0, ldc2, epilogue, alpha,
                      rowdot.data_ptr() if rowdot is not None else 0, rowdot_seg, rowdot_seq)
    N.check(N.lib.amdp_gemm(ctypes.byref(args), _stream()), "amdp_gemm")
    return C


def attention_fwd(qkv, batch, seq, heads, head_dim, causal=True, key_len=None):
    out = torch.empty(batch * seq, heads * head_dim, dtype=torch.bfloat16, device=qkv.device)
    lse = torch.empty(batch, heads, seq, dtype=torch.float32, device=qkv.device)
    N.check(N.lib.amdp_attention_fwd(_p(qkv), _p(out), _p(lse), batch, seq, heads, head_dim,
                                     int(causal), _p(key_len), _stream()), "amdp_attention_fwd")
    return out, lse


def attention_bwd(qkv, out, dout, lse, batch, seq, heads, head_dim, causal=True, key_len=None):
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(N.lib.amdp_attention_bwd_workspace(batch, seq, heads, head_dim),
                     dtype=torch.uint8, device=qkv.device)
    N.check(N.lib.amdp_attention_bwd(_p(qkv), _p(out), _p(dout), _p(lse), _p(dqkv), _p(ws),
                                     batch, seq, heads, head_dim, int(causal), _p(key_len), _stream()),
            "amdp_attention_bwd")
    return dqkv


def attention_bwd_delta(qkv, dout, lse, delta, batch, seq, heads, head_dim, causal=True, key_len=None,
                        scratch=True):
    """Backward with delta [batch][heads][seq] supplied.  scratch=True: amdp_attention_bwd_delta_ws
    (dK/dV store dS^T, dQ = dS K; the engine's path); False: amdp_attention_bwd_delta (the dQ
    kernel recomputes S / dP)."""
    dqkv = torch.empty_like(qkv)
    if scratch:
        ws = torch.empty(max(1, N.lib.amdp_attention_bwd_scratch_bytes(batch, seq, heads, head_dim, int(causal))),
                         dtype=torch.uint8, device=qkv.device)
        N.check(N.lib.amdp_attention_bwd_delta_ws(_p(qkv), _p(dout), _p(lse), _p(delta), _p(dqkv), _p(ws), batch, seq,
                                                  heads, head_dim, int(causal), _p(key_len), _stream()),
                "amdp_attention_bwd_delta_ws")
    else:
        N.check(N.lib.amdp_attention_bwd_delta(_p(qkv), _p(dout), _p(lse), _p(delta), _p(dqkv), batch, seq, heads,
                                               head_dim, int(causal), _p(key_len), _stream()), "amdp_attention_bwd_delta")
    return dqkv


def layernorm_fwd(x, gamma, beta, eps=1e-5):
    rows, cols = x.shape
    y = torch.empty_like(x)
    mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    rstd = torch.empty_like(mean)
    N.check(N.lib.amdp_layernorm_fwd(_p(x), _p(gamma), _p(beta), _p(y), _p(mean), _p(rstd),
                                     rows, cols, eps, _stream()), "amdp_layernorm_fwd")
    return y, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd, resid_grad, dgamma, dbeta):
    rows, cols = x.shape
    dx = torch.empty_like(x)
    ws = torch.empty(N.lib.amdp_layernorm_bwd_workspace(rows, cols), dtype=torch.uint8,
                     device=x.device)
    N.check(N.lib.amdp_layernorm_bwd(_p(dy), _p(x), _p(gamma), _p(mean), _p(rstd),
                                     _p(resid_grad), _p(dx), _p(dgamma), _p(dbeta), _p(ws),
                                     rows, cols, _stream()), "amdp_layernorm_bwd")
    return dx


def layernorm_bwd_parts(rows, cols):
    return N.lib.amdp_layernorm_bwd_parts(rows, cols)


def layernorm_bwd_rows(dy, x, gamma, mean, rstd, resid_grad, part):
    """dx, with the dgamma / dbeta column partials added into `part` (deferred form)."""
    rows, cols = x.shape
    dx = torch.empty_like(x)
    N.check(N.lib.amdp_layernorm_bwd_rows(_p(dy), _p(x), _p(gamma), _p(mean), _p(rstd), _p(resid_grad), _p(dx),
                                          _p(part), rows, cols, _stream()), "amdp_layernorm_bwd_rows")
    return dx


def layernorm_dgb_flush(part, nparts, cols, dgamma, dbeta):
    N.check(N.lib.amdp_layernorm_dgb_flush(_p(part), nparts, cols, _p(dgamma), _p(dbeta), _stream()),
            "amdp_layernorm_dgb_flush")


def embedding_fwd(tokens, wte, wpe, seq):
    ntok, hidden = tokens.numel(), wte.shape[1]
    x = torch.empty(ntok, hidden, dtype=torch.bfloat16, device=wte.device)
    N.check(N.lib.amdp_embedding_fwd(_p(tokens), _p(wte), _p(wpe), _p(x), ntok, seq, hidden,
                                     _stream()), "amdp_embedding_fwd")
    return x


def embedding_bwd(tokens, dx, dwte, dwpe, seq):
    ntok, hidden = dx.shape
    ws = torch.empty(ntok, dtype=torch.int32, device=dx.device)
    N.check(N.lib.amdp_embedding_bwd(_p(tokens), _p(dx), _p(dwte), _p(dwpe), _p(ws), ntok, seq, hidden,
                                     _stream()), "amdp_embedding_bwd")


def xent_fwd_bwd(logits, labels, loss_sum, scale):
    ntok, vocab = logits.shape
    rows = torch.empty(ntok, dtype=torch.float32, device=logits.device)
    N.check(N.lib.amdp_xent_fwd_bwd(_p(logits), _p(labels), _p(loss_sum), _p(rows), ntok, vocab,
                                    logits.stride(0), scale, _stream()), "amdp_xent_fwd_bwd")


def optimizer_step(kind, master, m, v, grad, w_bf16, *, lr, beta1=0.9, beta2=0.999, eps=1e-3,
                   weight_decay=0.0, clamp_min=1e-8, clamp_max=1e6, grad_scale=1.0, step=1):
    a = N.OptArgs(kind, lr, beta1, beta2, eps, weight_decay, clamp_min, clamp_max, grad_scale,
                  step)
    N.check(N.lib.amdp_optimizer_step(ctypes.byref(a), _p(master), _p(m), _p(v), _p(grad),
                                      _p(w_bf16), master.numel(), _stream()),
            "amdp_optimizer_step")


def fill_normal(n, seed, stddev, device="cuda"):
    w = torch.empty(n, dtype=torch.bfloat16, device=device)
    f = torch.empty(n, dtype=torch.float32, device=device)
    N.check(N.lib.amdp_fill_normal_bf16_f32(_p(w), _p(f), n, seed, stddev, _stream()),
            "amdp_fill_normal")
    return w, f
