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
