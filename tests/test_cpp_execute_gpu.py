"""A compiled C++ consumer of the drop-in API (tests/cpp/execute_tiny.cpp, linked against
libamdp.so) calls the reference's build/simulate and then ppsim::execute — the GPU
counterpart of simulate — on the tiny GPT config (D=4, 2 pipelines, 8 minibatches per window,
4 windows).  Checked against the reference fixture (tests/golden, from oracle/_ref) and the
CPU oracle replaying it: declared order = the reference timeline, measured per-device F/B
order = the reference's, GPU-observed versions bit-exact, losses within 1e-3, and the
reference audits pass on the measured Timeline."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def test_cpp_execute_matches_reference_and_oracle():
    import gpt_oracle as O

    cpp = os.path.join(ROOT, "tests", "cpp")
    subprocess.run(["make", "-C", cpp, "_build/execute_tiny"], check=True, capture_output=True)
    out = subprocess.run([os.path.join(cpp, "_build", "execute_tiny")], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    r = json.loads(out.stdout)
    cfg = ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 1]
    golden = next(e["csv"] for e in json.load(open(os.path.join(ROOT, "tests", "golden", "sched_golden.json")))
                  if e["config"] == cfg and "csv" in e)
    assert r["declared_csv"] == golden
    key = lambda rows: [",".join(x.split(",")[:7]) for x in rows.strip().split("\n")[1:]
                        if x.split(",")[1] in ("Forward", "Backward")]
    assert key(r["measured_csv"]) == key(golden)
    assert r["causality_issues"] == 0 and r["overlap_issues"] == 0 and r["max_mismatch"] <= 1

    inputs, labels = O.synthetic_tokens(64, 4, 1024, 1234, 0, 32)
    om = O.Model(4, 128, 4, 512, 1024, 64, 4, True, 1234)
    ol, _, seen = O.replay(golden, om, [1, 1, 1, 1], O.Opt("adamw", 1e-3, 0.9, 0.95, 1e-8, 0.0), 8, inputs, labels)
    for row in r["version_trace"].strip().split("\n")[1:]:
        dev, kind, stage, mb, pipe, w, pre, ver = row.split(",")
        assert int(ver) == seen[(kind, int(stage), int(mb))], row
    losses = np.array(r["losses"])
    assert np.max(np.abs(losses - ol) / np.abs(ol)) < 1e-3


def test_cpp_execute_two_ranks_on_one_gpu(tmp_path):
    """ppsim::execute with world_size 2 from C++ (ExecuteOptions::allgather over a shared
    directory), both ranks on one GPU through the peer-memory data plane: the union of the
    ranks' version traces and losses is the single-rank program's, to the bit (the fold puts
    every stage of the tiny D=4 config on one rank, so only stage-boundary hops cross)."""
    cpp = os.path.join(ROOT, "tests", "cpp")
    subprocess.run(["make", "-C", cpp, "_build/execute_tiny", "_build/execute_multirank"], check=True,
                   capture_output=True)
    one = json.loads(subprocess.run([os.path.join(cpp, "_build", "execute_tiny")], capture_output=True, text=True,
                                    timeout=600, check=True).stdout)
    procs = [subprocess.Popen([os.path.join(cpp, "_build", "execute_multirank"), str(r), "2", str(tmp_path)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600) for p in procs]
    assert all(p.returncode == 0 for p in procs), [o[1][-2000:] for o in outs]
    res = [json.loads(o[0]) for o in outs]
    losses = np.sum([np.array(r["losses"]) for r in res], axis=0)
    assert np.array_equal(losses.astype(np.float32), np.array(one["losses"], np.float32))
    rows = sorted(x for r in res for x in r["version_trace"].strip().split("\n")[1:])
    assert rows == sorted(one["version_trace"].strip().split("\n")[1:])
    assert all(r["p2p_bytes_sent"] > 0 and r["overlap_issues"] == 0 for r in res)
