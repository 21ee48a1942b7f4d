"""The drop-in boundary: libamdp.so loads without a GPU and exports every function the
C-ABI headers declare (include/amdp_kernels.h, amdp_sched.h, amdp_engine.h) and the C++
ppsim API entry points (include/ppsim/ppsim.hpp, execute.hpp).  No compute calls."""
import os
import re
import subprocess

from paper_2605_29664_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("amdp_kernels.h", "amdp_sched.h", "amdp_engine.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(amdp_[a-z0-9_]+)\s*\(", txt))
    return names


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(_native.lib, n)]
    assert not missing, missing


def test_cpp_api_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("build", "simulate", "bubble_ratio", "mismatch_report", "window_mismatch",
                "memory_report", "timeline_csv", "validate_cluster", "validate_policy",
                "validate_causality", "validate_non_overlap", "map_stage_to_device",
                "default_num_pipelines", "preload_count", "reduce_broadcast_cost", "execute"):
        assert re.search(r"ppsim::" + sym + r"(\[abi:cxx11\])?\(", out), sym


def test_version_string():
    assert _native.lib.amdp_version().decode().startswith("amdp-b200")


def test_attention_workspace_sizes():
    """Host-side sizing of the attention backward workspace (no device work): delta padded to
    256 B, then the dS^T scratch of the tiled kernels (one 16 KB chunk per 128-key tile and
    64-query half-block visited: causal n(n+1), bidirectional 2n^2 per sequence and head);
    the causal-agnostic size is the bidirectional upper bound; seq <= 128 (one-tile kernels)
    and head_dim 80 (dQ kernel recomputing S / dP) need no scratch."""
    L = _native.lib
    for B, S, H, D in [(4, 2048, 16, 128), (4, 1024, 16, 64), (4, 512, 16, 64), (2, 768, 3, 128)]:
        n = S // 128
        delta = (B * S * H * 4 + 255) // 256 * 256
        assert L.amdp_attention_bwd_scratch_bytes(B, S, H, D, 1) == B * H * n * (n + 1) * 16384
        assert L.amdp_attention_bwd_scratch_bytes(B, S, H, D, 0) == B * H * 2 * n * n * 16384
        assert L.amdp_attention_bwd_workspace_causal(B, S, H, D, 1) == delta + B * H * n * (n + 1) * 16384
        assert L.amdp_attention_bwd_workspace(B, S, H, D) == L.amdp_attention_bwd_workspace_causal(B, S, H, D, 0)
    assert L.amdp_attention_bwd_scratch_bytes(4, 64, 4, 32, 1) == 0
    assert L.amdp_attention_bwd_scratch_bytes(4, 2048, 32, 80, 1) == 0  # head_dim 80: recompute dQ kernel
    assert L.amdp_attention_bwd_workspace(4, 64, 4, 32) == 4 * 64 * 4 * 4
