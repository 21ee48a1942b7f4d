"""The multi-rank data plane, executed: N ranks (one process each) sharing ONE B200 through the
executor's CUDA-IPC peer-memory backend (paper_2605_29664_b200/csrc/engine/comm_ipc.cu), the
same code that moves stage-boundary activations / gradients and the window Reduce / Broadcast /
all-reduce between GPUs of an NVLink box.  Every run is compared with the single-rank run of
the same configuration:

  * N=2, AMDP ZeRO: the fold within replica groups puts every stage on one rank, so only
    stage-boundary hops cross ranks -> losses and final weights are BIT-IDENTICAL to N=1
    (every kernel is deterministic: no atomics in the stage math, fixed-order reductions);
  * N=4, AMDP ZeRO: every stage spans 2 ranks -> Reduce to the owner + bf16/LayerNorm
    broadcast run for real; the gradient sum associates differently from N=1's single
    buffer, so losses / weights match within float rounding (stated below);
  * N=4, AMDP replicated (ZeRO off): the window all-reduce (reduce-scatter + all-gather over
    peer memory) at the first Update(w, i, .);
  * N=2, DAPPLE; N=2 on the production attention shapes (head_dim 64).

In every case the per-task parameter versions equal the reference's (the union of the ranks'
version traces is the N=1 trace, which test_engine_gpu.py pins to the oracle) and each rank's
dispatch order is its part of the reference timeline.  Two consecutive runs are made so the
epoch-valued flags are exercised across runs.
"""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

# name: (model, depth, threshold, windows, schedule, zero)
CASES = {
    "tiny_d4_zero": ("tiny", 4, 8, 3, "AMDP", True),
    "tiny_d4_replicated": ("tiny", 4, 8, 3, "AMDP", False),
    "tiny_d4_dapple": ("tiny", 4, 8, 2, "DAPPLE", False),
    "hd64_d4_zero": ("hd64", 4, 8, 2, "AMDP", True),
}


def _model(name):
    from paper_2605_29664_b200 import engine as E
    if name == "tiny":
        m = E.ModelConfig.tiny()
        m.layers_per_stage = [1, 1, 1, 1]
    else:
        m = E.ModelConfig(4, 512, 8, 2048, 2048, 256)
        m.layers_per_stage = [1, 1, 1, 1]
    return m


def _run_case(case, world, rank, allgather):
    from paper_2605_29664_b200 import engine as E
    mname, depth, thr, windows, schedule, zero = CASES[case]
    model = _model(mname)
    run = E.RunConfig(depth=depth, threshold=thr, windows=windows, schedule=schedule, zero=zero,
                      world_size=world, rank=rank,
                      optimizer=E.OptimizerConfig(kind=3, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0))
    eng = E.Engine(model, run, allgather=allgather)
    init = {s["stage"]: eng.stage_params(s["stage"]) for s in eng.plan()["stages"] if s["hosted"]}
    inputs, labels = E.synthetic_tokens(model, run.data_seed, 0, run.num_minibatches)
    l1 = eng.run(inputs, labels).copy()
    l2 = eng.run(inputs, labels).copy()  # continue training: second epoch of every flag
    plan = eng.plan()
    # fp32 masters this rank is authoritative for: a whole stage (single-rank group) or its
    # ZeRO shard (ranges) of a stage shared by several ranks
    owned = {}
    for s in plan["stages"]:
        if s["owner"]:
            owned[s["stage"]] = (eng.stage_params(s["stage"]), s["shard"])
    rows = eng.version_trace().strip().split("\n")[1:]
    st = eng.stats()
    last = any(s["hosted"] and s["stage"] == depth - 1 for s in plan["stages"])
    out = dict(losses=(l1, l2) if last else None, owned=owned, init=init, rows=rows, plan=plan, stats=st)
    eng.close()
    return out


def _worker(case, world, rank, port, outdir):
    import pickle

    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_29664_b200 import engine as E
    try:
        res = _run_case(case, world, rank, E.torch_allgather())
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(res, f)
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(case, world, tmp_path):
    import pickle

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(case, world, r, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [pickle.load(open(os.path.join(tmp_path, f"r{r}.pkl"), "rb")) for r in range(world)]


@pytest.fixture(scope="module")
def single_rank():
    cache = {}

    def get(case):
        if case not in cache:
            cache[case] = _run_case(case, 1, 0, None)
        return cache[case]
    return get


def _merge(results):
    # a minibatch's loss is reported by the rank that ran its last-stage forward (0 elsewhere)
    have = [r["losses"] for r in results if r["losses"] is not None]
    losses = tuple(np.sum([h[k] for h in have], axis=0) for k in (0, 1))
    owned, covered = {}, {}
    for r in results:
        for st, (vals, shard) in r["owned"].items():
            if not shard:
                owned[st] = vals
                covered[st] = np.ones(vals.size, bool)
                continue
            dst = owned.setdefault(st, np.zeros_like(vals))
            cov = covered.setdefault(st, np.zeros(vals.size, bool))
            for lo, hi in shard:
                dst[lo:hi] = vals[lo:hi]
                cov[lo:hi] = True
    for st, cov in covered.items():  # the shards tile the parameters (alignment padding aside)
        assert cov.mean() > 0.99, (st, cov.mean())
    rows = sorted(row for r in results for row in r["rows"])
    return losses, owned, rows


@pytest.mark.parametrize("case,world,exact", [
    ("tiny_d4_zero", 2, True),
    ("tiny_d4_zero", 4, False),
    ("tiny_d4_replicated", 4, False),
    ("tiny_d4_dapple", 2, True),
    ("hd64_d4_zero", 2, True),
])
def test_ranks_on_one_gpu_match_single_rank(case, world, exact, single_rank, tmp_path):
    ref = single_rank(case)
    res = _launch(case, world, tmp_path)
    losses, owned, rows = _merge(res)
    # the data plane actually moved data between the ranks
    assert sum(r["stats"]["p2p_bytes_sent"] for r in res) > 0
    if not exact:
        assert sum(r["stats"]["collective_bytes"] for r in res) > 0
        assert res[0]["plan"]["collectives"] > 0
    # version trace: bit-exact union of the ranks' traces
    assert rows == sorted(ref["rows"])
    depth = CASES[case][1]
    assert set(owned) == set(range(depth))
    for k in (0, 1):
        a, b = np.asarray(losses[k], np.float64), np.asarray(ref["losses"][k], np.float64)
        if exact:
            assert np.array_equal(a, b), (k, np.max(np.abs(a - b)))
        else:
            # different association of the fp32 window-gradient sum only (observed ~1e-6)
            assert np.max(np.abs(a - b) / np.abs(b)) < 1e-4
    for i in range(depth):
        a, b = owned[i].astype(np.float64), ref["owned"][i][0].astype(np.float64)
        if exact:
            assert np.array_equal(a, b), (i, np.max(np.abs(a - b)))
        else:
            # Adam divides by sqrt(v): a gradient entry that nearly cancels across replicas keeps
            # only rounding noise, which the update normalises to a full step; bound the error
            # against the update itself as the oracle tests do (test_engine_gpu.py)
            upd = np.linalg.norm(b - ref["init"][i].astype(np.float64))
            assert np.linalg.norm(a - b) / np.linalg.norm(b) < 2e-3, (i, np.linalg.norm(a - b) / np.linalg.norm(b))
            assert np.linalg.norm(a - b) / upd < 5e-2, (i, np.linalg.norm(a - b) / upd)
