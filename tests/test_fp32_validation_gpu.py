"""fp32 validation mode (north_star: "tightened for an fp32 validation mode").

ModelConfig.fp32_validation runs every stage in fp32 end to end (amdp_f32_* kernels: fp32
activations, weights read from the fp32 master, fp32 accumulation, tanhf / expf / logf) on the
same executor, schedule and version semantics as the bf16 production path.  Against the CPU
oracle replaying the reference trace WITHOUT bf16 rounding (fp64 math, emulate_bf16=False) the
per-minibatch losses and final weights then agree to float rounding:

  losses       : relative error < 2e-5   (bf16 mode: 1e-3)
  final weights: ||dw|| / ||w|| < 2e-5, and < 2e-3 of the update itself
                 (bf16 mode: 5e-3 and 8e-2)

Schedules: AMDP ZeRO declared 1:1 (preload 1) and the reference's canonical 1:2 (preload 2)
with the reference AdamType rule (optim.hpp:256-266) under replicated updates.
"""
import json
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))

LOSS_RTOL = 2e-5
WEIGHT_RTOL = 2e-5
UPDATE_RTOL = 2e-3

MODELS = {
    # name: (layers, hidden, heads, ffn, vocab, seq)
    "tiny": (4, 128, 4, 512, 1024, 64),
    "hd64": (4, 512, 8, 2048, 2048, 256),
    "bert_pad": (4, 128, 4, 512, 1024, 64),  # bidirectional MLM, padded sequences (pad id 7)
}
PAD = {"bert_pad": 7}
OPTS = {
    "adamw": (3, dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8), ("adamw", 1e-3, 0.9, 0.95, 1e-8, 0.0)),
    "adamtype": (2, dict(lr=2e-4, beta1=0.9, beta2=0.999, eps=1e-3), ("adamtype", 2e-4, 0.9, 0.999, 1e-3, 0.0)),
}
# name: (model, threshold, windows, declared bwd, zero, optimizer)
CASES = {
    "tiny_preload1_zero_adamw": ("tiny", 8, 3, 1, True, "adamw"),
    "tiny_preload2_replicated_adamtype": ("tiny", 8, 3, 2, False, "adamtype"),
    "hd64_preload1_zero_adamw": ("hd64", 8, 3, 1, True, "adamw"),
    "bert_pad_preload1_zero_adamw": ("bert_pad", 8, 3, 1, True, "adamw"),
}


def _golden_csv(cfg):
    for e in json.load(open(os.path.join(HERE, "golden", "sched_golden.json"))):
        if e["config"] == cfg and "csv" in e:
            return e["csv"]
    raise KeyError(cfg)


@pytest.fixture(scope="module", params=list(CASES))
def f32_run(request):
    from fractions import Fraction

    import gpt_oracle as O
    from paper_2605_29664_b200 import engine as E
    mname, thr, windows, bwd, zero, oname = CASES[request.param]
    L, h, H, f, V, S = MODELS[mname]
    pad = PAD.get(mname, 0)
    model = E.ModelConfig(L, h, H, f, V, S, causal=not pad, pad_token=pad)
    model.layers_per_stage = [1, 1, 1, 1]
    model.fp32_validation = True
    kind, kw, okw = OPTS[oname]
    run = E.RunConfig(depth=4, threshold=thr, windows=windows, declared_bwd=Fraction(bwd), zero=zero,
                      optimizer=E.OptimizerConfig(kind=kind, weight_decay=0.0, **kw))
    eng = E.Engine(model, run)
    init = [eng.stage_params(i) for i in range(4)]
    inputs, labels = E.synthetic_tokens(model, run.data_seed, 0, run.num_minibatches)
    losses = eng.run(inputs, labels)
    final = [eng.stage_params(i) for i in range(4)]
    trace = _golden_csv(["AMDP", 4, 4, "1", str(bwd), "0", "0", 2, 2, thr, thr * windows, int(zero)])
    om = O.Model(L, h, H, f, V, S, 4, not pad, model.seed, pad_token=pad)
    ol, omaster, seen = O.replay(trace, om, [1, 1, 1, 1], O.Opt(*okw), thr, inputs, labels, emulate_bf16=False)
    out = dict(eng=eng, init=init, final=final, losses=losses, ol=ol, omaster=omaster, seen=seen, O=O)
    yield out
    eng.close()


def test_fp32_losses_match_fp64_oracle(f32_run):
    gl, ol = f32_run["losses"], f32_run["ol"]
    rel = np.abs(gl - ol) / np.abs(ol)
    assert rel.max() < LOSS_RTOL, rel.max()


def test_fp32_versions_bit_exact(f32_run):
    rows = f32_run["eng"].version_trace().strip().split("\n")[1:]
    for r in rows:
        _, kind, stage, mb, *_rest, ver = r.split(",")
        assert int(ver) == f32_run["seen"][(kind, int(stage), int(mb))], r


def test_fp32_final_weights_match_fp64_oracle(f32_run):
    O = f32_run["O"]
    plan = f32_run["eng"].plan()
    for i in range(4):
        st = plan["stages"][i]
        ref = O.flat_stage(f32_run["omaster"][i], st["params"], st["numel"])
        got = f32_run["final"][i].astype(np.float64)
        upd = np.linalg.norm(ref - f32_run["init"][i].astype(np.float64))
        err = np.linalg.norm(got - ref)
        assert upd > 0
        assert err / np.linalg.norm(ref) < WEIGHT_RTOL, (i, err / np.linalg.norm(ref))
        assert err / upd < UPDATE_RTOL, (i, err / upd)


@pytest.mark.parametrize("a_mn,b_mn,epi", [(False, False, 0), (True, True, 3), (False, True, 4), (False, False, 1),
                                           (False, False, 2)])
def test_f32_gemm_matches_torch(a_mn, b_mn, epi):
    """amdp_f32_gemm in every layout / epilogue the fp32 stage uses, against torch fp64."""
    import ctypes

    from paper_2605_29664_b200 import _native as N
    torch.manual_seed(11)
    M, N_, K = 200, 136, 88  # ragged: not multiples of the 64-wide tiles
    A = torch.randn(M, K, device="cuda", dtype=torch.float64)
    B = torch.randn(N_, K, device="cuda", dtype=torch.float64)
    acc = A @ B.T
    aux = torch.randn(M, N_, device="cuda", dtype=torch.float64)
    C0 = torch.randn(M, N_, device="cuda", dtype=torch.float64)
    k0, k1 = 0.7978845608028654, 0.044715
    gelu = lambda x: 0.5 * x * (1 + torch.tanh(k0 * x * (1 + k1 * x * x)))  # noqa: E731
    t = torch.tanh(k0 * aux * (1 + k1 * aux * aux))
    dgelu = 0.5 * (1 + t) + 0.5 * aux * (1 - t * t) * k0 * (1 + 3 * k1 * aux * aux)
    want = {0: acc, 1: gelu(acc), 2: acc + aux, 3: C0 + acc, 4: acc * dgelu}[epi]
    Af = (A.T.contiguous() if a_mn else A).float()
    Bf = (B.T.contiguous() if b_mn else B).float()
    C = (C0.float().clone() if epi == 3 else torch.zeros(M, N_, device="cuda"))
    C2 = torch.zeros(M, N_, device="cuda")
    auxf = aux.float()
    args = N.GemmArgs(M, N_, K, Af.data_ptr(), M if a_mn else K, int(a_mn), Bf.data_ptr(), N_ if b_mn else K,
                      int(b_mn), C.data_ptr(), N_, auxf.data_ptr(), N_, C2.data_ptr(), N_, epi, 1.0, 0, 0, 0)
    N.check(N.lib.amdp_f32_gemm(ctypes.byref(args), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
            "amdp_f32_gemm")
    torch.cuda.synchronize()
    assert torch.allclose(C.double(), want, rtol=1e-4, atol=1e-4)
    if epi == 1:
        assert torch.allclose(C2.double(), acc, rtol=1e-5, atol=1e-4)
