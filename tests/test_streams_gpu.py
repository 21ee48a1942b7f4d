"""Concurrent compute streams on one GPU (executor.cu: plan_streams): each logical device's
tasks run in order on their own stream, tasks of different devices overlap.  The cross-stream
waits cover every shared resource and a stage's backwards keep their global order, so the run
must be BIT-IDENTICAL to the single-stream executor (AMDP_SINGLE_STREAM=1): losses, fp32
master weights, per-task versions — eagerly and as a replayed CUDA graph — and the measured
timeline must keep one task at a time per logical device (the reference's audits).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(kind, single, monkeypatch):
    from paper_2605_29664_b200 import engine as E
    if single:
        monkeypatch.setenv("AMDP_SINGLE_STREAM", "1")
    else:
        monkeypatch.delenv("AMDP_SINGLE_STREAM", raising=False)
    if kind == "tiny_d4":
        m, depth = E.ModelConfig.tiny(), 4
        m.layers_per_stage = [1, 1, 1, 1]
    elif kind == "hd64_d4":
        m, depth = E.ModelConfig(4, 512, 8, 2048, 2048, 256), 4
        m.layers_per_stage = [1, 1, 1, 1]
    elif kind == "wide_d4":  # 1.3B-wide layers (h 2048, ffn 8192, head_dim 128): CTA-pair GEMMs with
        # N-split tails and K-split weight-gradient tails (per-stream flag buffers), tcgen05 attention
        m, depth = E.ModelConfig(4, 2048, 16, 8192, 4096, 512), 4
        m.layers_per_stage = [1, 1, 1, 1]
    else:  # BERT-like, D=8: 8 concurrent streams, bidirectional MLM
        m, depth = E.ModelConfig(8, 256, 4, 1024, 2048, 128, causal=False), 8
        m.layers_per_stage = [1] * 8
    run = E.RunConfig(depth=depth, threshold=2 * depth, windows=3,
                      optimizer=E.OptimizerConfig(kind=3, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0))
    eng = E.Engine(m, run)
    toks = E.PinnedTokens(run.num_minibatches, m.tokens_per_minibatch)
    E.synthetic_tokens(m, run.data_seed, 0, run.num_minibatches, out=toks)
    out = []
    for _ in range(3):  # eager, captured, replayed
        eng.run_windows(run.windows, toks.inputs, toks.labels, toks.losses)
        out.append((toks.losses.copy(), eng.version_trace(), eng.stats()["graph_replayed"]))
    rep = eng.timeline().report(run.policy(), warmup=0)
    w = [eng.stage_params(i) for i in range(depth)]
    streams = eng.plan()["compute_streams"]
    eng.close()
    return out, w, rep, streams


@pytest.mark.parametrize("kind", ["tiny_d4", "hd64_d4", "wide_d4", "bert_d8"])
def test_concurrent_streams_bit_identical_to_single_stream(kind, monkeypatch):
    multi, wm, rep, ns = _run(kind, False, monkeypatch)
    single, ws, _, ns1 = _run(kind, True, monkeypatch)
    assert ns1 == 1 and ns == (8 if kind == "bert_d8" else 4)
    assert [o[2] for o in multi] == [0, 1, 1]
    for (la, ta, _), (lb, tb, _) in zip(multi, single):
        assert np.array_equal(la, lb)
        assert ta == tb
    for a, b in zip(wm, ws):
        assert np.array_equal(a, b)
    assert rep["causality_issues"] == [] and rep["overlap_issues"] == []
