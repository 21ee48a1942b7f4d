"""Python host mirror of the AMDP-B200 executor (include/amdp_engine.h).

    eng = Engine(ModelConfig.gpt_1p3b(), RunConfig(depth=8, threshold=32, windows=10))
    losses = eng.run(inputs, labels)          # host token arrays (pinned), one schedule pass
    tl = eng.timeline()                       # measured ppsim Timeline (same type as simulate())
    ppsim.bubble_ratio(tl, 1)

Everything executes inside libamdp.so; there is no CPU or eager-PyTorch fallback.
"""
from __future__ import annotations

import ctypes
import json
from ctypes import (POINTER, Structure, byref, c_char_p, c_double, c_float, c_int, c_int64,
                    c_size_t, c_uint8, c_uint64, c_void_p)
from dataclasses import dataclass, field
from fractions import Fraction
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from . import ppsim as P

lib = N.lib


class _Model(Structure):
    _fields_ = [("layers", c_int), ("hidden", c_int), ("heads", c_int), ("ffn", c_int),
                ("vocab", c_int), ("seq", c_int), ("seqs_per_minibatch", c_int),
                ("causal", c_int), ("init_std", c_float), ("ln_eps", c_float),
                ("seed", c_uint64), ("layers_per_stage", POINTER(c_int)), ("recompute", c_int),
                ("fp32_validation", c_int), ("pad_token", c_int)]


class _Run(Structure):
    _fields_ = [("policy", P._Policy), ("declared_fwd", P._Rat), ("declared_bwd", P._Rat),
                ("optimizer", N.OptArgs), ("world_size", c_int), ("rank", c_int),
                ("record_events", c_int), ("data_seed", c_uint64), ("plan_only", c_int),
                ("depth", c_int), ("comm_backend", c_int)]

COMM_IPC, COMM_NCCL = 0, 1


class _Stats(Structure):
    _fields_ = [("device_ms", c_double), ("tasks_executed", c_int64), ("kernels_launched", c_int64),
                ("h2d_bytes", c_int64), ("d2h_bytes", c_int64), ("p2p_bytes_sent", c_int64),
                ("collective_bytes", c_int64), ("busy_ms", c_double),
                ("host_issue_ms", c_double), ("graph_replayed", c_int64)]


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype, f.argtypes = res, args


_sig("amdp_nccl_unique_id", c_int, [POINTER(c_uint8)])
_sig("amdp_engine_create", c_void_p, [POINTER(_Model), POINTER(_Run), POINTER(c_uint8), c_char_p, c_size_t])
_sig("amdp_engine_destroy", None, [c_void_p])
_sig("amdp_host_alloc", c_void_p, [c_size_t])
_sig("amdp_host_free", None, [c_void_p])
_sig("amdp_synthetic_tokens", c_int, [POINTER(_Model), c_uint64, c_int, c_int, c_void_p, c_void_p])
_sig("amdp_engine_run", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_char_p, c_size_t])
_sig("amdp_engine_stats", c_int, [c_void_p, POINTER(_Stats)])
_sig("amdp_engine_run_windows", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int, c_char_p, c_size_t])
_sig("amdp_engine_stage_tokens", c_int, [c_void_p, c_void_p, c_void_p])
_sig("amdp_engine_set_kernel_timing", c_int, [c_void_p, c_int])
_sig("amdp_engine_set_graphs", c_int, [c_void_p, c_int])
_sig("amdp_engine_set_streams", c_int, [c_void_p, c_int])


class _KStat(Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("launches", c_int64), ("total_ms", c_double),
                ("flops", c_double), ("bytes", c_double)]


_sig("amdp_engine_kernel_stats", c_int, [c_void_p, POINTER(_KStat), c_int])
_sig("amdp_engine_num_events", c_int, [c_void_p])
_sig("amdp_engine_events", c_int, [c_void_p, POINTER(P._Event), c_int])
_sig("amdp_engine_num_lane_events", c_int, [c_void_p])
_sig("amdp_engine_lane_events", c_int, [c_void_p, POINTER(P._Event), c_int])
_sig("amdp_engine_version_trace", c_size_t, [c_void_p, c_char_p, c_size_t])
_sig("amdp_engine_schedule", c_void_p, [c_void_p])
_sig("amdp_engine_stage_numel", c_int64, [c_void_p, c_int])
_sig("amdp_engine_get_stage_params", c_int, [c_void_p, c_int, c_void_p, c_int64])
_sig("amdp_engine_set_stage_params", c_int, [c_void_p, c_int, c_void_p, c_int64])
_sig("amdp_engine_plan_json", c_size_t, [c_void_p, c_char_p, c_size_t])
_sig("amdp_engine_comm_export", c_size_t, [c_void_p, c_void_p, c_size_t])
_sig("amdp_engine_comm_connect", c_int, [c_void_p, POINTER(c_void_p), POINTER(c_size_t), c_int, c_char_p, c_size_t])


@dataclass
class ModelConfig:
    layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    seq: int
    seqs_per_minibatch: int = 4   # the paper's microbatch size
    causal: bool = True
    init_std: float = 0.02
    ln_eps: float = 1e-5
    seed: int = 1234
    layers_per_stage: Optional[List[int]] = None
    recompute: bool = False  # backward rebuilds f = gelu(u) and o = attention(qkv) (amdp_model_config)
    fp32_validation: bool = False  # every tensor / product fp32 on the CUDA cores (amdp_f32_* kernels)
    pad_token: int = 0  # bidirectional models: token id (> 0) marking padding; 0 = no padding

    @property
    def tokens_per_minibatch(self) -> int:
        return self.seq * self.seqs_per_minibatch

    def flops_per_token(self) -> float:
        """Training FLOPs per token, 6 L (4h^2 + 2 h ffn) + 12 L s h + 6 h V."""
        L, h, s, V, f = self.layers, self.hidden, self.seq, self.vocab, self.ffn
        return 6 * L * (4 * h * h + 2 * h * f) + 12 * L * s * h + 6 * h * V

    @staticmethod
    def tiny():
        return ModelConfig(4, 128, 4, 512, 1024, 64)

    @staticmethod
    def gpt_350m():
        return ModelConfig(24, 1024, 16, 4096, 50304, 1024)

    @staticmethod
    def bert_large():
        return ModelConfig(24, 1024, 16, 4096, 30528, 512, causal=False)

    @staticmethod
    def gpt_1p3b():
        return ModelConfig(24, 2048, 16, 8192, 50304, 2048)

    @staticmethod
    def gpt_2p7b():
        return ModelConfig(32, 2560, 32, 10240, 50304, 2048)

    def _c(self):
        lps = None
        if self.layers_per_stage:
            lps = (c_int * len(self.layers_per_stage))(*self.layers_per_stage)
        m = _Model(self.layers, self.hidden, self.heads, self.ffn, self.vocab, self.seq,
                   self.seqs_per_minibatch, int(self.causal), self.init_std, self.ln_eps,
                   self.seed, lps, int(self.recompute), int(self.fp32_validation), int(self.pad_token))
        m._keep = lps
        return m


@dataclass
class OptimizerConfig:
    kind: int = N.OPT_ADAMW
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0
    clamp_min: float = 1e-8
    clamp_max: float = 1e6
    grad_scale: float = 1.0

    def _c(self):
        return N.OptArgs(self.kind, self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                         self.clamp_min, self.clamp_max, self.grad_scale, 1)


@dataclass
class RunConfig:
    depth: int
    threshold: int
    windows: int
    declared_fwd: Fraction = Fraction(1)
    declared_bwd: Fraction = Fraction(1)   # uniform 1:1 -> preload 1 (SURVEY §7 hard part 1)
    optimizer: OptimizerConfig = field(default_factory=OptimizerConfig)
    world_size: int = 1
    rank: int = 0
    record_events: bool = True
    data_seed: int = 1234
    plan_only: bool = False   # host-side plan without CUDA/NCCL (multi-rank tests on CPU)
    # "AMDP" (d/2 pipelines; ZeRO Reduce/Broadcast unless zero=False: replicated per-pipeline
    # Update), "Chimera" (two bidirectional pipelines, replicated), the synchronous
    # single-pipeline baselines "DAPPLE" / "GPipe", "Interleaved1F1B" (two stage chunks per
    # device: depth = 2 x devices) and "PipeDreamAsync" (an update after every backward);
    # builder.hpp:145-338 for each policy's tasks and dependencies.
    schedule: str = "AMDP"
    zero: bool = True
    # world_size > 1: "ipc" (this library's CUDA-IPC peer-memory data plane; also runs
    # several ranks on one GPU) or "nccl"
    comm: str = "ipc"

    @property
    def num_minibatches(self) -> int:
        return self.windows * self.threshold

    def policy(self) -> P.PolicyConfig:
        M = self.num_minibatches
        if self.schedule == "AMDP":
            return P.PolicyConfig(P.Policy.AMDP, 2, self.depth // 2, self.threshold, M, bool(self.zero))
        if self.schedule in ("DAPPLE", "GPipe", "Interleaved1F1B"):
            return P.PolicyConfig(P.Policy[self.schedule], self.threshold, 1, self.threshold, M, False)
        if self.schedule == "Chimera":
            return P.PolicyConfig(P.Policy.Chimera, self.threshold, 2, self.threshold, M, False)
        if self.schedule == "PipeDreamAsync":
            return P.PolicyConfig(P.Policy.PipeDreamAsync, min(self.depth, self.threshold), 1,
                                  self.threshold, M, False)
        raise ValueError(f"unknown schedule {self.schedule!r}")

    @property
    def devices(self) -> int:
        return self.depth // 2 if self.schedule == "Interleaved1F1B" else self.depth

    def declared_cluster(self) -> P.ClusterSpec:
        return P.ClusterSpec.uniform(self.depth, self.devices, self.declared_fwd, self.declared_bwd)

    def _c(self):
        return _Run(self.policy()._c(), P._r(self.declared_fwd), P._r(self.declared_bwd),
                    self.optimizer._c(), self.world_size, self.rank, int(self.record_events),
                    self.data_seed, int(self.plan_only), self.depth,
                    COMM_NCCL if self.comm == "nccl" else COMM_IPC)


def torch_allgather(group=None):
    """An `allgather` for Engine over an initialised torch.distributed process group."""
    import torch.distributed as dist

    def gather(blob: bytes):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, blob, group=group)
        return out
    return gather


def nccl_unique_id() -> bytes:
    buf = (c_uint8 * 128)()
    N.check(lib.amdp_nccl_unique_id(buf), "amdp_nccl_unique_id")
    return bytes(buf)


class PinnedTokens:
    """Pinned host arrays inputs/labels [M][T] int32 and losses [M] float32 (cudaHostAlloc
    through the C-ABI): copies overlap compute, and runs over them can be CUDA graphs."""

    def __init__(self, num_minibatches: int, tokens: int):
        n = num_minibatches * tokens * 4
        self._pi = lib.amdp_host_alloc(n)
        self._pl = lib.amdp_host_alloc(n)
        if not self._pi or not self._pl:
            raise MemoryError("cudaHostAlloc failed")
        self.inputs = np.ctypeslib.as_array((ctypes.c_int32 * (num_minibatches * tokens)).from_address(self._pi)).reshape(num_minibatches, tokens)
        self.labels = np.ctypeslib.as_array((ctypes.c_int32 * (num_minibatches * tokens)).from_address(self._pl)).reshape(num_minibatches, tokens)
        self._ps = lib.amdp_host_alloc(num_minibatches * 4)
        if not self._ps:
            raise MemoryError("cudaHostAlloc failed")
        self.losses = np.ctypeslib.as_array((ctypes.c_float * num_minibatches).from_address(self._ps))

    def __del__(self):
        if lib is None:  # interpreter teardown: the process exit releases the pinned pages
            return
        for p in (getattr(self, "_pi", None), getattr(self, "_pl", None), getattr(self, "_ps", None)):
            if p:
                lib.amdp_host_free(p)


def synthetic_tokens(model: ModelConfig, data_seed: int, first: int, count: int, out=None):
    T = model.tokens_per_minibatch
    if out is None:
        inputs = np.empty((count, T), np.int32)
        labels = np.empty((count, T), np.int32)
    else:
        inputs, labels = out.inputs[first:first + count], out.labels[first:first + count]
    N.check(lib.amdp_synthetic_tokens(byref(model._c()), data_seed, first, count,
                                      inputs.ctypes.data, labels.ctypes.data), "amdp_synthetic_tokens")
    return inputs, labels


class Engine:
    """One rank of the executor.  world_size > 1: pass `allgather` (bytes -> list of every
    rank's bytes, in rank order; e.g. `torch_allgather` over torch.distributed) so the
    ranks exchange their communication descriptors (IPC backend), or `nccl_id` for NCCL."""

    def __init__(self, model: ModelConfig, run: RunConfig, nccl_id: Optional[bytes] = None,
                 allgather=None):
        self.model, self.runcfg = model, run
        err = ctypes.create_string_buffer(4096)
        idb = (c_uint8 * 128)(*nccl_id) if nccl_id else None
        self._m, self._r = model._c(), run._c()
        h = lib.amdp_engine_create(byref(self._m), byref(self._r), idb, err, len(err))
        if not h:
            raise RuntimeError("amdp_engine_create: " + err.value.decode())
        self._h = h
        if run.world_size > 1 and not run.plan_only and run.comm != "nccl":
            if allgather is None:
                raise ValueError("world_size > 1 with the IPC backend needs an allgather callable")
            self.connect(allgather(self.comm_descriptor()))

    def comm_descriptor(self) -> bytes:
        n = lib.amdp_engine_comm_export(self._h, None, 0)
        buf = ctypes.create_string_buffer(max(1, n))
        lib.amdp_engine_comm_export(self._h, buf, n)
        return buf.raw[:n]

    def connect(self, descriptors: Sequence[bytes]) -> None:
        bufs = [ctypes.create_string_buffer(bytes(d), max(1, len(d))) for d in descriptors]
        ptrs = (c_void_p * len(bufs))(*[ctypes.cast(b, c_void_p) for b in bufs])
        lens = (c_size_t * len(bufs))(*[len(d) for d in descriptors])
        err = ctypes.create_string_buffer(4096)
        if lib.amdp_engine_comm_connect(self._h, ptrs, lens, len(bufs), err, len(err)) != 0:
            raise RuntimeError("amdp_engine_comm_connect: " + err.value.decode())

    def close(self):
        if getattr(self, "_h", None):
            lib.amdp_engine_destroy(self._h)
            self._h = None

    __del__ = close

    def run(self, inputs: np.ndarray, labels: np.ndarray, losses: Optional[np.ndarray] = None) -> np.ndarray:
        M = self.runcfg.num_minibatches
        assert inputs.shape == (M, self.model.tokens_per_minibatch) and inputs.dtype == np.int32
        if losses is None:
            losses = np.zeros(M, np.float32)
        err = ctypes.create_string_buffer(4096)
        rc = lib.amdp_engine_run(self._h, inputs.ctypes.data, labels.ctypes.data, losses.ctypes.data,
                                 err, len(err))
        if rc != 0:
            raise RuntimeError("amdp_engine_run: " + err.value.decode())
        return losses

    def run_windows(self, num_windows: int, inputs: np.ndarray, labels: np.ndarray,
                    losses: Optional[np.ndarray] = None, resident: bool = False) -> np.ndarray:
        """Windows [0, num_windows) of the schedule, pipeline starting empty (one bench 'run')."""
        if losses is None:
            losses = np.zeros(self.runcfg.num_minibatches, np.float32)
        err = ctypes.create_string_buffer(4096)
        rc = lib.amdp_engine_run_windows(self._h, num_windows, inputs.ctypes.data, labels.ctypes.data,
                                         losses.ctypes.data, int(resident), err, len(err))
        if rc != 0:
            raise RuntimeError("amdp_engine_run_windows: " + err.value.decode())
        return losses

    def stage_tokens(self, inputs: np.ndarray, labels: np.ndarray) -> None:
        N.check(lib.amdp_engine_stage_tokens(self._h, inputs.ctypes.data, labels.ctypes.data),
                "amdp_engine_stage_tokens")

    def set_kernel_timing(self, on: bool) -> None:
        lib.amdp_engine_set_kernel_timing(self._h, int(on))

    def set_streams(self, n: int) -> int:
        """Concurrent compute streams in use (1 = serial executor); returns the count."""
        r = lib.amdp_engine_set_streams(self._h, int(n))
        if r < 0:
            raise RuntimeError("amdp_engine_set_streams failed")
        return r

    def set_graphs(self, on: bool) -> None:
        """CUDA graphs of whole runs (default on, one GPU; needs pinned host buffers)."""
        lib.amdp_engine_set_graphs(self._h, int(on))

    def kernel_stats(self) -> dict:
        arr = (_KStat * 16)()
        n = lib.amdp_engine_kernel_stats(self._h, arr, 16)
        return {a.name.decode(): dict(launches=a.launches, ms=a.total_ms, flops=a.flops, bytes=a.bytes)
                for a in arr[:n]}

    def stats(self) -> dict:
        s = _Stats()
        lib.amdp_engine_stats(self._h, byref(s))
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    def timeline(self) -> P.Timeline:
        n = lib.amdp_engine_num_events(self._h)
        arr = (P._Event * max(1, n))()
        lib.amdp_engine_events(self._h, arr, n)
        evs = [P.TaskEvent(P.Kind(e.kind), e.stage, e.minibatch, e.pipeline, e.device,
                           P._f(e.start), P._f(e.duration), bool(e.preloaded), e.window) for e in arr[:n]]
        rc = self.runcfg
        return P.Timeline.from_events(evs, rc.policy().policy, rc.depth, rc.devices, rc.threshold,
                                      rc.declared_cluster())

    def lane_events(self) -> list:
        """Reduce / Broadcast intervals on the collective / update streams (see timeline())."""
        n = lib.amdp_engine_num_lane_events(self._h)
        arr = (P._Event * max(1, n))()
        lib.amdp_engine_lane_events(self._h, arr, n)
        return [P.TaskEvent(P.Kind(e.kind), e.stage, e.minibatch, e.pipeline, e.device,
                            P._f(e.start), P._f(e.duration), bool(e.preloaded), e.window) for e in arr[:n]]

    def declared_timeline(self) -> P.Timeline:
        h = P._Handle(lib.amdp_engine_schedule(self._h))
        n = P.lib.amdp_schedule_num_tasks(h.h)
        arr = (c_int * max(1, n))()
        P.lib.amdp_schedule_order(h.h, arr, n)
        rc = self.runcfg
        return P.Timeline(h, rc.policy().policy, rc.depth, rc.devices, rc.threshold, rc.declared_cluster(),
                          list(arr[:n]))

    def version_trace(self) -> str:
        n = lib.amdp_engine_version_trace(self._h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib.amdp_engine_version_trace(self._h, buf, n + 1)
        return buf.raw[:n].decode()

    def plan(self) -> dict:
        n = lib.amdp_engine_plan_json(self._h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib.amdp_engine_plan_json(self._h, buf, n + 1)
        return json.loads(buf.value.decode())

    def stage_params(self, stage: int) -> np.ndarray:
        n = lib.amdp_engine_stage_numel(self._h, stage)
        out = np.empty(n, np.float32)
        N.check(lib.amdp_engine_get_stage_params(self._h, stage, out.ctypes.data, n), "get_stage_params")
        return out

    def set_stage_params(self, stage: int, values: np.ndarray) -> None:
        v = np.ascontiguousarray(values, np.float32)
        N.check(lib.amdp_engine_set_stage_params(self._h, stage, v.ctypes.data, v.size), "set_stage_params")
