"""ctypes binding to libamdp.so (the C-ABI in include/amdp_kernels.h, include/amdp_sched.h,
include/amdp_engine.h).

There is deliberately no fallback: if the shared library is missing the import fails
loudly, so no test or benchmark can silently run a CPU or eager-PyTorch path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int, c_int32, c_int64,
                    c_size_t, c_uint16, c_uint64, c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
# AMDP_LIB: an alternative in-tree build (A/B timing of two library versions on one box).
LIB_PATH = os.environ.get("AMDP_LIB") or os.path.join(_HERE, "libamdp.so")


class NativeLibraryMissing(RuntimeError):
    pass


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    return ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)


lib = _load()

# ------------------------------------------------------------------ kernels
EPI_STORE_BF16, EPI_GELU, EPI_RESIDUAL, EPI_ACCUM_F32, EPI_GELU_BWD, EPI_STORE_F32, EPI_ROWDOT = range(7)
OPT_SGD, OPT_MOMENTUM, OPT_REF_ADAMTYPE, OPT_ADAMW = range(4)
ATTN_IMPL_MMA_SYNC, ATTN_IMPL_TCGEN05 = range(2)


class GemmArgs(Structure):
    _fields_ = [("M", c_int), ("N", c_int), ("K", c_int),
                ("A", c_void_p), ("lda", c_int), ("a_mn_major", c_int),
                ("B", c_void_p), ("ldb", c_int), ("b_mn_major", c_int),
                ("C", c_void_p), ("ldc", c_int),
                ("aux", c_void_p), ("ld_aux", c_int),
                ("C2", c_void_p), ("ldc2", c_int),
                ("epilogue", c_int), ("alpha", c_float),
                ("rowdot", c_void_p), ("rowdot_seg", c_int), ("rowdot_seq", c_int)]


class OptArgs(Structure):
    _fields_ = [("kind", c_int), ("lr", c_float), ("beta1", c_float), ("beta2", c_float),
                ("eps", c_float), ("weight_decay", c_float), ("clamp_min", c_float),
                ("clamp_max", c_float), ("grad_scale", c_float), ("step", c_int)]


def _sig(name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


_P = c_void_p
_sig("amdp_gemm", c_int, [POINTER(GemmArgs), _P])
_sig("amdp_f32_gemm", c_int, [POINTER(GemmArgs), _P])
_sig("amdp_attention_fwd", c_int, [_P, _P, _P, c_int, c_int, c_int, c_int, c_int, _P, _P])
_sig("amdp_attention_bwd_workspace", c_size_t, [c_int, c_int, c_int, c_int])
_sig("amdp_attention_bwd", c_int,
     [_P, _P, _P, _P, _P, _P, c_int, c_int, c_int, c_int, c_int, _P, _P])
_sig("amdp_attention_bwd_delta_supported", c_int, [c_int, c_int])
_sig("amdp_attention_impl", c_int, [c_int, c_int, c_int])
_sig("amdp_gelu_fwd", c_int, [_P, _P, c_int64, _P])
_sig("amdp_attention_bwd_delta", c_int,
     [_P, _P, _P, _P, _P, c_int, c_int, c_int, c_int, c_int, _P, _P])
_sig("amdp_attention_bwd_delta_ws", c_int,
     [_P, _P, _P, _P, _P, _P, c_int, c_int, c_int, c_int, c_int, _P, _P])
_sig("amdp_attention_bwd_workspace_causal", c_size_t, [c_int, c_int, c_int, c_int, c_int])
_sig("amdp_attention_bwd_scratch_bytes", c_size_t, [c_int, c_int, c_int, c_int, c_int])
_sig("amdp_layernorm_fwd", c_int, [_P, _P, _P, _P, _P, _P, c_int, c_int, c_float, _P])
_sig("amdp_layernorm_bwd_workspace", c_size_t, [c_int, c_int])
_sig("amdp_layernorm_bwd", c_int,
     [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int, c_int, _P])
_sig("amdp_layernorm_bwd_parts", c_int, [c_int, c_int])
_sig("amdp_layernorm_bwd_rows", c_int, [_P, _P, _P, _P, _P, _P, _P, _P, c_int, c_int, _P])
_sig("amdp_layernorm_dgb_flush", c_int, [_P, c_int, c_int, _P, _P, _P])
_sig("amdp_embedding_fwd", c_int, [_P, _P, _P, _P, c_int, c_int, c_int, _P])
_sig("amdp_embedding_bwd", c_int, [_P, _P, _P, _P, _P, c_int, c_int, c_int, _P])
_sig("amdp_xent_fwd_bwd", c_int, [_P, _P, _P, _P, c_int, c_int, c_int, c_float, _P])
_sig("amdp_optimizer_step", c_int, [POINTER(OptArgs), _P, _P, _P, _P, _P, c_int64, _P])
_sig("amdp_sumsq", c_int, [_P, c_int64, _P, _P])
_sig("amdp_fill_normal_bf16_f32", c_int, [_P, _P, c_int64, c_uint64, c_float, _P])
_sig("amdp_fill_const_f32", c_int, [_P, c_int64, c_float, _P])
_sig("amdp_version", c_char_p, [])


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed with code {rc}")
