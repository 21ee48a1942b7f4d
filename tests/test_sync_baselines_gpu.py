"""The reference's other schedules executed by the same GPU stage executor as AMDP (ZeRO):
the synchronous baselines DAPPLE / GPipe (one pipeline, per-window Update), Interleaved1F1B
(two stage chunks per device), Chimera and AMDP without ZeRO (two / d/2 pipelines with
replicated per-pipeline Updates, builder.hpp:306-336) and PipeDreamAsync (an Update after
every backward).  Checked like the AMDP run in test_engine_gpu.py: the executor replays the
reference's dispatch order, the GPU-observed version trace is bit-exact with the one the CPU
oracle derives from the UNMODIFIED reference's timeline (tests/golden), and the per-minibatch
losses match the oracle's replay of that trace.  Tiny GPT, D=4, 8 minibatches per window, 4
windows, all logical devices folded on one B200."""
import json
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
LOSS_RTOL = 1e-3  # north_star: 1e-3 in bf16 compute with fp32 accumulation


def _golden_csv(cfg):
    for e in json.load(open(os.path.join(HERE, "golden", "sched_golden.json"))):
        if e["config"] == cfg and "csv" in e:
            return e["csv"]
    raise KeyError(cfg)


GOLDEN = {
    ("DAPPLE", True): ["DAPPLE", 4, 4, "1", "1", "0", "0", 8, 1, 8, 32, 0],
    ("GPipe", True): ["GPipe", 4, 4, "1", "1", "0", "0", 8, 1, 8, 32, 0],
    ("Interleaved1F1B", True): ["Interleaved1F1B", 4, 2, "1", "1", "0", "0", 8, 1, 8, 32, 0],
    ("Chimera", True): ["Chimera", 4, 4, "1", "1", "0", "0", 8, 2, 8, 32, 0],
    ("AMDP", False): ["AMDP", 4, 4, "1", "1", "0", "0", 2, 2, 8, 32, 0],
    ("PipeDreamAsync", True): ["PipeDreamAsync", 4, 4, "1", "1", "0", "0", 4, 1, 8, 32, 0],
}
SYNCHRONOUS = ("DAPPLE", "GPipe", "Interleaved1F1B", "Chimera")


@pytest.mark.parametrize("schedule,zero", list(GOLDEN), ids=lambda x: str(x))
def test_schedule_matches_reference_trace(schedule, zero):
    import gpt_oracle as O
    from paper_2605_29664_b200 import engine as E
    from paper_2605_29664_b200 import ppsim as P

    model = E.ModelConfig.tiny()
    model.layers_per_stage = [1, 1, 1, 1]
    opt = E.OptimizerConfig(kind=3, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
    run = E.RunConfig(depth=4, threshold=8, windows=4, optimizer=opt, schedule=schedule, zero=zero)
    eng = E.Engine(model, run)
    init = [eng.stage_params(i) for i in range(4)]
    inputs, labels = E.synthetic_tokens(model, run.data_seed, 0, run.num_minibatches)
    losses = eng.run(inputs, labels)

    trace = _golden_csv(GOLDEN[(schedule, zero)])
    assert P.timeline_csv(eng.declared_timeline()) == trace  # the executor replays the reference order
    om = O.Model(4, 128, 4, 512, 1024, 64, 4, True, model.seed)
    div = 1 if schedule == "PipeDreamAsync" else 8
    ol, omaster, seen = O.replay(trace, om, [1, 1, 1, 1], O.Opt("adamw", 1e-3, 0.9, 0.95, 1e-8, 0.0), 8, inputs, labels,
                           update_div=div)
    rel = np.max(np.abs(losses - ol) / np.abs(ol))
    assert rel < LOSS_RTOL, rel
    rows = eng.version_trace().strip().split("\n")[1:]
    assert len(rows) == 2 * 4 * run.num_minibatches
    bad = [r for r in rows if int(r.split(",")[-1]) != seen[(r.split(",")[1], int(r.split(",")[2]), int(r.split(",")[3]))]]
    assert not bad, bad[:3]
    if schedule in SYNCHRONOUS:  # every Forward / Backward of window w reads version w
        for r in rows:
            f = r.split(",")
            assert int(f[-1]) == int(f[5]), r
    tl = eng.timeline()
    assert P.validate_non_overlap(tl) == []
    # final weights (every replica holds the same values): same tolerances as the AMDP run
    plan = eng.plan()
    for i in range(4):
        st = plan["stages"][i]
        ref = O.flat_stage(omaster[i], st["params"], st["numel"])
        got = eng.stage_params(i).astype(np.float64)
        upd = np.linalg.norm(ref - init[i].astype(np.float64))
        err = np.linalg.norm(got - ref)
        assert upd > 0
        # PipeDreamAsync takes 8x the optimizer steps, each on one minibatch's gradient: more
        # bf16 rounding enters the weights (1e-2 instead of 5e-3)
        wtol = 1e-2 if schedule == "PipeDreamAsync" else 5e-3
        assert err / np.linalg.norm(ref) < wtol, (i, err / np.linalg.norm(ref), err / upd)
        assert err / upd < 6e-2, (i, err / upd)
