"""The CPU oracle is pinned before it is trusted (CPU-only tests).

  * update rule: oracle.gpt_oracle.apply_update vs the reference's own
    ppsim::detail::apply_update run on seeded vectors (tests/golden/optim_golden.json,
    generated from the unmodified reference by tests/golden/make_optim_golden.py), and the
    reference's closed-form iterates (T/test_optim.cpp:34-53);
  * schedule: the oracle replays the reference trace; its derived versions equal the
    structural law F = w - preloaded, B = w (builder.hpp:289-304);
  * synthetic data / init generators are deterministic and seed-sensitive.
"""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
import gpt_oracle as O  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "optim_golden.json")))
SCHED = json.load(open(os.path.join(HERE, "golden", "sched_golden.json")))


def _kind(name):
    return {"sgd": "sgd", "momentum": "momentum"}.get(name, "adamtype")


@pytest.mark.parametrize("case", GOLD, ids=lambda c: c["name"])
def test_apply_update_matches_reference(case):
    opt = O.Opt(_kind(case["name"]), case["eta"], case["beta1"], case["beta2"], case["epsilon"], 0.0,
                case["clamp_min"], case["clamp_max"])
    th = np.array(case["theta0"], np.float64)
    m, v = np.zeros_like(th), np.zeros_like(th)
    for step, (g, want) in enumerate(zip(case["grads"], case["iterates"]), 1):
        O.apply_update(opt, th, m, v, np.array(g, np.float64), step)
        np.testing.assert_allclose(th, want, rtol=0, atol=1e-14)


def test_closed_form_sgd_iterates():  # T/test_optim.cpp:34-53: F = x^2/2, eta 0.1
    opt = O.Opt("sgd", 0.1)
    th = np.array([1.0])
    seq = [1.0]
    for _ in range(3):
        O.apply_update(opt, th, None, None, th.copy(), 1)
        seq.append(th[0])
    assert np.allclose(seq, [1, 0.9, 0.81, 0.729], atol=1e-15)
    # one-step delay: gradient of the previous iterate
    th, prev, seq = np.array([1.0]), np.array([1.0]), [1.0]
    for t in range(3):
        g = (prev if t >= 1 else th).copy()
        prev = th.copy()
        O.apply_update(opt, th, None, None, g, 1)
        seq.append(th[0])
    assert np.allclose(seq, [1, 0.9, 0.8, 0.71], atol=1e-15)


def test_replay_versions_follow_structural_law():
    e = [x for x in SCHED if x["config"] == ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 1]][0]
    ev = O.parse_timeline_csv(e["csv"])
    ev.sort(key=lambda x: (x["start"], x["dur"] > 0, x["device"], x["row"]))
    ver = [0] * 4
    for x in ev:
        if x["kind"] == "Broadcast":
            ver[x["stage"]] += 1
        elif x["kind"] == "Forward":
            assert ver[x["stage"]] == x["window"] - x["preloaded"]
        elif x["kind"] == "Backward":
            assert ver[x["stage"]] == x["window"]


def test_generators_deterministic():
    a = O.synthetic_tokens(64, 4, 1024, 7, 0, 3)
    b = O.synthetic_tokens(64, 4, 1024, 7, 0, 3)
    c = O.synthetic_tokens(64, 4, 1024, 8, 0, 3)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert not np.array_equal(a[0], c[0])
    assert np.array_equal(a[1][:, :-1].reshape(-1)[:63], a[0][:, 1:].reshape(-1)[:63])  # next-token labels
    w = O.normal_init(100000, 5, 0.02)
    assert abs(w.std() - 0.02) < 5e-4 and abs(w.mean()) < 5e-4


def test_bf16_rounding_is_nearest_even():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5, 3.14159], np.float32)
    r = O.bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == np.float32(1.0 + 2 ** -7)
    assert r[3] == -2.5


EXEC_CONFIGS = [
    ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 1],
    ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 0],
    ["Chimera", 4, 4, "1", "1", "0", "0", 8, 2, 8, 32, 0],
    ["DAPPLE", 4, 4, "1", "1", "0", "0", 8, 1, 8, 32, 0],
    ["GPipe", 4, 4, "1", "1", "0", "0", 8, 1, 8, 32, 0],
    ["Interleaved1F1B", 4, 2, "1", "1", "0", "0", 8, 1, 8, 32, 0],
    ["PipeDreamAsync", 4, 4, "1", "1", "0", "0", 4, 1, 8, 32, 0],
]


@pytest.mark.parametrize("cfg", EXEC_CONFIGS, ids=lambda c: f"{c[0]}-zero{c[-1]}")
def test_replay_versions_match_reference_mismatch_report(cfg):
    """The replay's per-replica versions (Broadcast rewrites every replica of a stage, Update
    only its own pipeline's) reproduce the reference's own mismatch_report: updates between
    F finish and B start per (stage, minibatch) (analysis.hpp:28-88, fixture from the
    unmodified reference)."""
    e = [x for x in SCHED if x["config"] == cfg][0]
    m = O.Model(4, 32, 2, 64, 64, 16, 1, True, 3)
    M = cfg[10]
    inputs, labels = O.synthetic_tokens(16, 1, 64, 1234, 0, M)
    div = 1 if cfg[0] == "PipeDreamAsync" else cfg[9]
    losses, _, seen = O.replay(e["csv"], m, [1, 1, 1, 1], O.Opt("adamw", 1e-3, 0.9, 0.95, 1e-8, 0.0),
                               cfg[9], inputs, labels, update_div=div)
    assert np.all(np.isfinite(losses))
    nz = {(s, j): n for s, j, n in e["mismatch_nonzero"]}
    for i in range(4):
        for j in range(M):
            assert seen[("Backward", i, j)] - seen[("Forward", i, j)] == nz.get((i, j), 0), (i, j)
