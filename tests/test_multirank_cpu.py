"""Multi-GPU host logic on CPU: the per-rank plans of the executor (plan_only engines; no
CUDA/NCCL) for world sizes 2/4/8 folding the D=8 logical devices of the 1.3B headline
config.  Checked: every logical device / stage is hosted where map_stage_to_device puts it
(H/builder.hpp:81-88), each rank's NCCL program pairs up exactly with its peers' (same
positions in the global dispatch order), collectives are issued by exactly the stage's
replica group, and the joint communication program cannot deadlock under rendezvous
semantics.  A world_size-2 gloo job runs the same check through torch.distributed."""
import os
import sys

import pytest

from paper_2605_29664_b200 import engine as E
from paper_2605_29664_b200 import ppsim as P


def _plans(world, windows=2, depth=8, thr=32):
    model = E.ModelConfig.gpt_1p3b()
    out = []
    for r in range(world):
        run = E.RunConfig(depth=depth, threshold=thr, windows=windows, world_size=world, rank=r,
                          plan_only=True)
        out.append(E.Engine(model, run).plan())
    return out


def _check(plans, depth=8):
    world = len(plans)
    fold = plans[0]["device_rank"]
    for r, pl in enumerate(plans):
        assert pl["device_rank"] == fold
        hosted = {s["stage"] for s in pl["stages"] if s["hosted"]}
        want = {i for i in range(depth) for p in range(depth // 2)
                if fold[P.map_stage_to_device(p, i, depth)] == r}
        assert hosted == want
        for s in pl["stages"]:
            assert s["owner_rank"] == fold[s["stage"]]  # the reference's owner: the rank of device i
            grp = sorted({fold[P.map_stage_to_device(p, s["stage"], depth)] for p in range(depth // 2)})
            assert s["group"] == grp
            # ZeRO within a multi-rank replica group: every member keeps the optimizer state of
            # its shard (1/|group| of every segment); a single-rank group's rank keeps all of it
            if len(grp) > 1:
                assert s["owner"] == s["hosted"]
                if s["hosted"]:
                    assert s["shard"] and abs(s["opt_numel"] * len(grp) / s["numel"] - 1) < 0.01
            else:
                assert s["owner"] == (fold[s["stage"]] == r) and s["shard"] == []
    # p2p pairing (message ids agree), collectives issued by exactly the replica group
    ops = [[tuple(o) for o in pl["comm_ops"]] for pl in plans]
    for r in range(world):
        for (k, kind, peer, stage, mid) in ops[r]:
            if kind == "send":
                assert (k, "recv", r, -1, mid) in ops[peer], (r, k, peer)
            elif kind == "recv":
                assert (k, "send", r, -1, mid) in ops[peer], (r, k, peer)
            else:
                members = plans[r]["stages"][stage]["group"]
                for m in members:
                    assert (k, kind, -1, stage, mid) in ops[m]
    # rendezvous simulation of the joint program (NCCL backend: one stream per rank)
    pos = [0] * world
    while True:
        progressed = False
        for r in range(world):
            if pos[r] >= len(ops[r]):
                continue
            k, kind, peer, stage, mid = ops[r][pos[r]]
            if kind in ("send", "recv"):
                if pos[peer] < len(ops[peer]):
                    k2, kind2, peer2, _, mid2 = ops[peer][pos[peer]]
                    if k2 == k and peer2 == r and kind2 != kind and mid2 == mid:
                        pos[r] += 1
                        pos[peer] += 1
                        progressed = True
            else:
                members = plans[r]["stages"][stage]["group"]
                if all(pos[m] < len(ops[m]) and ops[m][pos[m]] == (k, kind, -1, stage, mid) for m in members):
                    for m in members:
                        pos[m] += 1
                    progressed = True
        if all(pos[r] >= len(ops[r]) for r in range(world)):
            return sum(len(o) for o in ops)
        assert progressed, f"communication deadlock at positions {pos}"


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_plans_pair_and_cannot_deadlock(world):
    n = _check(_plans(world))
    if world == 1:
        assert n == 0  # all replicas co-resident: no traffic at all
    else:
        assert n > 0


@pytest.mark.parametrize("world,fold,hosted,group_size", [
    (1, [0] * 8, [set(range(8))], 1),
    # components of map_stage_to_device at d=8: {0,3,4,7} and {1,2,5,6} (H/builder.hpp:81-88)
    (2, [0, 1, 1, 0, 0, 1, 1, 0], [{0, 3, 4, 7}, {1, 2, 5, 6}], 1),
    (4, [0, 2, 2, 0, 1, 3, 3, 1], [{0, 3, 4, 7}, {0, 3, 4, 7}, {1, 2, 5, 6}, {1, 2, 5, 6}], 2),
    (8, list(range(8)), None, 4),
])
def test_fold_within_replica_groups(world, fold, hosted, group_size):
    """Logical devices fold onto ranks within replica groups: at N=2 every stage lives on one
    GPU (no collective at all), at N=4 every stage spans 2 ranks, at N=8 its 4 devices."""
    plans = _plans(world)
    assert plans[0]["device_rank"] == fold
    for r, pl in enumerate(plans):
        if hosted is not None:
            assert {s["stage"] for s in pl["stages"] if s["hosted"]} == hosted[r]
        for s in pl["stages"]:
            assert len(s["group"]) == group_size
        # per stage and window: one Reduce + one Broadcast per parameter segment (embeddings /
        # layer / head), 2 windows
        segs = sum(1 + n + (s == 0) + (s == 7) for s, n in enumerate(pl["partition"]))
        assert pl["collectives"] == (0 if group_size == 1 else 2 * segs)
        kinds = {o[1] for o in pl["comm_ops"]}
        if world == 2:
            assert kinds == {"send", "recv"}


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model = E.ModelConfig.gpt_1p3b()
    run = E.RunConfig(depth=8, threshold=32, windows=2, world_size=world, rank=rank, plan_only=True)
    mine = E.Engine(model, run).plan()
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    if rank == 0:
        try:
            q.put(("ok", _check(allp)))
        except AssertionError as e:  # pragma: no cover
            q.put(("fail", str(e)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_plans_consistent():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    status, val = q.get(timeout=10)
    assert status == "ok", val
    assert val > 0


@pytest.mark.parametrize("schedule", ["DAPPLE", "GPipe"])
@pytest.mark.parametrize("world", [1, 2, 4])
def test_synchronous_baselines_plan(schedule, world):
    """DAPPLE / GPipe on the executor (one pipeline, stage i on device i, per-window Update):
    every stage is hosted and owned by the rank of its device, replica groups are single
    ranks (no collectives), and the P2P program pairs up across ranks."""
    model = E.ModelConfig.gpt_1p3b()
    plans = []
    for r in range(world):
        run = E.RunConfig(depth=8, threshold=8, windows=2, world_size=world, rank=r, plan_only=True,
                          schedule=schedule)
        plans.append(E.Engine(model, run).plan())
    per = 8 // world
    fold = plans[0]["device_rank"]
    assert fold == [d // per for d in range(8)]  # no shared stages: contiguous fold
    for r, pl in enumerate(plans):
        for s in pl["stages"]:
            assert s["hosted"] == (s["stage"] // per == r)
            assert s["owner"] == (s["stage"] // per == r)
            assert s["group"] == [s["stage"] // per]
        assert all(o[1] in ("send", "recv") for o in pl["comm_ops"])
    ops = [[tuple(o) for o in pl["comm_ops"]] for pl in plans]
    for r in range(world):
        for (k, kind, peer, stage, mid) in ops[r]:
            assert (k, "recv" if kind == "send" else "send", r, -1, mid) in ops[peer]


@pytest.mark.parametrize("schedule,zero", [("AMDP", False), ("Chimera", False)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_replicated_update_plans(schedule, zero, world):
    """Replicated-update schedules with several pipelines (AMDP with ZeRO off, Chimera;
    builder.hpp:306-336): every rank hosting a replica of stage i keeps its own optimizer state,
    the window gradient is all-reduced over the stage's replica group at the first
    Update(w, i, .) of the global order (issued by exactly the group, same position on every
    member), and the joint P2P + collective program cannot deadlock."""
    model = E.ModelConfig.gpt_1p3b()
    thr = 8 if schedule == "Chimera" else 32
    plans = []
    for r in range(world):
        run = E.RunConfig(depth=8, threshold=thr, windows=2, world_size=world, rank=r, plan_only=True,
                          schedule=schedule, zero=zero)
        plans.append(E.Engine(model, run).plan())
    fold = plans[0]["device_rank"]
    if schedule == "Chimera":
        dev = lambda p, i: i if p == 0 else 7 - i  # noqa: E731  (builder.hpp:160)
        pipes = 2
    else:
        dev = lambda p, i: P.map_stage_to_device(p, i, 8)  # noqa: E731
        pipes = 4
    for r, pl in enumerate(plans):
        for s in pl["stages"]:
            grp = sorted({fold[dev(p, s["stage"])] for p in range(pipes)})
            assert s["group"] == grp
            assert s["hosted"] == (r in grp)
            assert s["owner"] == s["hosted"]  # replicated optimizer state
        kinds = {o[1] for o in pl["comm_ops"]}
        assert kinds <= {"send", "recv", "allreduce"}
    ops = [[tuple(o) for o in pl["comm_ops"]] for pl in plans]
    if world == 1:
        assert not any(ops[0])
        return
    n_ar = sum(o[1] == "allreduce" for o in ops[0])
    hosted0 = [s for s in plans[0]["stages"] if s["hosted"] and len(s["group"]) > 1]
    assert n_ar == 2 * len(hosted0)  # one per window per multi-rank hosted stage
    assert _check_joint(plans) > 0


def _check_joint(plans):
    """Pairing + rendezvous simulation of the joint program (any collective kinds)."""
    world = len(plans)
    ops = [[tuple(o) for o in pl["comm_ops"]] for pl in plans]
    for r in range(world):
        for (k, kind, peer, stage, mid) in ops[r]:
            if kind in ("send", "recv"):
                assert (k, "recv" if kind == "send" else "send", r, -1, mid) in ops[peer]
            else:
                for m in plans[r]["stages"][stage]["group"]:
                    assert (k, kind, -1, stage, mid) in ops[m]
    pos = [0] * world
    while not all(pos[r] >= len(ops[r]) for r in range(world)):
        progressed = False
        for r in range(world):
            if pos[r] >= len(ops[r]):
                continue
            k, kind, peer, stage, mid = ops[r][pos[r]]
            if kind in ("send", "recv"):
                if pos[peer] < len(ops[peer]) and ops[peer][pos[peer]] == (k, "recv" if kind == "send" else "send", r, -1, mid):
                    pos[r] += 1
                    pos[peer] += 1
                    progressed = True
            else:
                members = plans[r]["stages"][stage]["group"]
                if all(pos[m] < len(ops[m]) and ops[m][pos[m]] == (k, kind, -1, stage, mid) for m in members):
                    for m in members:
                        pos[m] += 1
                    progressed = True
        assert progressed, f"communication deadlock at positions {pos}"
    return sum(len(o) for o in ops)


@pytest.mark.parametrize("schedule", ["Interleaved1F1B", "PipeDreamAsync"])
def test_single_pipeline_schedules_plan(schedule):
    """Interleaved1F1B folds stage chunks i and i + devices onto device i (builder.hpp:165);
    PipeDreamAsync updates after every backward.  One replica per stage: no collectives."""
    model = E.ModelConfig.gpt_1p3b()
    plans = []
    for r in range(2):
        run = E.RunConfig(depth=8, threshold=8, windows=2, world_size=2, rank=r, plan_only=True,
                          schedule=schedule)
        plans.append(E.Engine(model, run).plan())
    devices = 4 if schedule == "Interleaved1F1B" else 8
    per = devices // 2
    for r, pl in enumerate(plans):
        for s in pl["stages"]:
            d = s["stage"] % devices
            assert s["hosted"] == (d // per == r)
            assert s["group"] == [d // per]
        assert all(o[1] in ("send", "recv") for o in pl["comm_ops"])
    assert _check_joint(plans) > 0


def test_unsupported_schedules_rejected():
    model = E.ModelConfig.tiny()
    with pytest.raises(ValueError):
        E.Engine(model, E.RunConfig(depth=4, threshold=8, windows=2, plan_only=True, schedule="ZeroBubble"))
    with pytest.raises(RuntimeError):  # AMDP needs an even depth (validate.hpp:60-73)
        E.Engine(model, E.RunConfig(depth=3, threshold=8, windows=2, plan_only=True))


@pytest.mark.parametrize("zero", [True, False])
def test_memory_accounting_matches_reference_model(zero):
    """what each rank of the 8-GPU 1.3B run allocates, in the units of the
    reference's memory_report (H/analysis.hpp:226-330) on the same schedule: stage replicas
    (weights), gradient buffers, optimizer-state multiples (ZeRO: 2 x replicas x 2/d) and live
    activations.  The executor frees an activation slot at its backward's position in the
    dispatch order, so it never needs more than the reference's closed-interval peak."""
    model = E.ModelConfig.gpt_1p3b()
    for r in range(8):
        run = E.RunConfig(depth=8, threshold=32, windows=2, world_size=8, rank=r, plan_only=True, zero=zero)
        eng = E.Engine(model, run)
        mem = eng.plan()["memory"]
        ref = P.memory_report(eng.declared_timeline(), run.policy())["per_device"][r]
        assert mem["weight_units"] == ref["weight"] == 4
        assert mem["gradient_units"] == ref["gradient"]
        # ZeRO: the owner's m, v for one stage = 4 replicas x 2 x 2/8; replicated: every replica
        assert mem["optimizer_state_units"] == ref["optimizer_state"] == (2 if zero else 8)
        assert 0 < mem["activation_slots"] <= ref["activation_peak"]
        parts = [k for k in mem if k not in ("total", "measured_device_bytes") and not k.endswith(("_units", "_slots"))]
        assert mem["total"] == sum(mem[k] for k in parts)
        assert mem["total"] < 180e9  # fits one B200's HBM


def test_recompute_fits_2p7b_d8_on_one_gpu():
    """GPT-2.7B D=8 folded on one GPU: 224 GB planned with stored activations, under the
    B200's 180 GB once f and o are recomputed (5 of 16 h-widths per layer and slot)."""
    m = E.ModelConfig.gpt_2p7b()
    full = E.Engine(m, E.RunConfig(depth=8, threshold=32, windows=2, plan_only=True)).plan()["memory"]
    m.recompute = True
    rc = E.Engine(m, E.RunConfig(depth=8, threshold=32, windows=2, plan_only=True)).plan()["memory"]
    assert full["total"] > 180e9 > rc["total"]
    assert rc["activations"] < full["activations"] * 0.72
