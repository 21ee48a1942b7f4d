"""CUDA graphs of whole runs (executor.cu: Engine::run / issue).

After one eager run, each new run configuration (windows, resident, host buffers, loss scales)
is captured once and replayed — the multi-stream program with its events, PDL edges, copies and
the K-split GEMMs' completion flags (which reset themselves, so a replay starts clean).  Every
kernel is deterministic, so an engine replaying graphs must produce the SAME BITS as an engine
issuing eagerly: losses, fp32 master weights, the per-task version trace; and the replayed
timeline (external event-record nodes) must pass the reference's audits.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _engine(kind):
    from paper_2605_29664_b200 import engine as E
    if kind == "tiny_gpt":
        m = E.ModelConfig.tiny()
    elif kind == "tiny_bert":  # bidirectional MLM: per-minibatch loss scales differ
        m = E.ModelConfig(4, 128, 4, 512, 1024, 64, causal=False)
    else:  # production kernels: tcgen05 attention head_dim 64, pair GEMMs
        m = E.ModelConfig(4, 512, 8, 2048, 2048, 256)
    m.layers_per_stage = [1, 1, 1, 1]
    run = E.RunConfig(depth=4, threshold=8, windows=3,
                      optimizer=E.OptimizerConfig(kind=3, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0))
    return E, m, run


@pytest.mark.parametrize("kind", ["tiny_gpt", "tiny_bert", "hd64"])
def test_graph_replay_is_bit_identical_to_eager(kind):
    from paper_2605_29664_b200 import ppsim as P
    E, model, run = _engine(kind)
    toks = E.PinnedTokens(run.num_minibatches, model.tokens_per_minibatch)
    E.synthetic_tokens(model, run.data_seed, 0, run.num_minibatches, out=toks)
    res = {}
    for graphs in (False, True):
        eng = E.Engine(model, run)
        eng.set_graphs(graphs)
        out = []
        for r in range(4):
            resident = r == 3  # a second configuration: captured on its first run
            if resident:
                eng.stage_tokens(toks.inputs, toks.labels)
            eng.run_windows(run.windows, toks.inputs, toks.labels, toks.losses, resident=resident)
            st = eng.stats()
            out.append(dict(losses=toks.losses.copy(), graph=st["graph_replayed"], trace=eng.version_trace(),
                            launches=st["kernels_launched"], tl=eng.timeline()))
        out.append([eng.stage_params(i) for i in range(4)])
        res[graphs] = out
        if graphs:
            tl = out[2]["tl"]
            rep = tl.report(run.policy(), warmup=0)
            assert rep["causality_issues"] == [] and rep["overlap_issues"] == []
            assert len(tl.flat()) == len(out[0]["tl"].flat()) and P.bubble_ratio(tl, 0) < 1
        eng.close()
    eager, graph = res[False], res[True]
    assert [o["graph"] for o in eager[:4]] == [0, 0, 0, 0]
    assert [o["graph"] for o in graph[:4]] == [0, 1, 1, 1]  # run 1 eager, then captured / replayed
    for a, b in zip(eager[:4], graph[:4]):
        assert np.array_equal(a["losses"], b["losses"])
        assert a["trace"] == b["trace"]
        assert a["launches"] == b["launches"]
    for wa, wb in zip(eager[4], graph[4]):
        assert np.array_equal(wa, wb)
