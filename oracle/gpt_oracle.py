"""CPU oracle for the AMDP training path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference legs may
import this module, and only as the checker or the timed CPU baseline; the product path
(paper_2605_29664_b200/) never imports it.

What it restates, and how it is pinned:
  * The schedule / version semantics come from the UNMODIFIED reference: the trace replayed
    here is the reference's own timeline_csv (oracle/_ref/ppsim_ref, or the committed
    fixture tests/golden/sched_golden.json generated from it).  Events are applied in time
    order; Broadcast(w, i) rewrites stage i (analysis.hpp:20-26, 47-52), so a Forward reads
    the number of stage-i broadcasts finished by its start and a Backward likewise — the
    mismatch semantics of analysis.hpp:28-88 (no weight stash; a preloaded minibatch's
    backward uses the new weights with its old activations, builder.hpp:289-304).
  * The update rule restates ppsim::detail::apply_update (optim.hpp:234-268) for the
    reference AdamType / SGD / Momentum kinds (pinned by tests/test_oracle.py against the
    reference's closed-form iterates, T/test_optim.cpp:34-53), plus AdamW.
  * PARITY UNPINNED for the network arithmetic: the reference has no model;
    the GPT stage math below (pre-LN, tanh-GELU, causal attention, untied head, no linear
    biases) defines the contract the GPU kernels are checked against, with bf16 rounding
    emulated at the points where the GPU stores bf16 (emulate_bf16=True).
"""
from __future__ import annotations

import csv
import io
import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

M64 = (1 << 64) - 1

# Elementwise passes over [T, ffn] activations dominate the replay time; numpy ufuncs release
# the GIL, so they run chunked over the host's cores (the matmuls are already threaded BLAS).
_NT = max(1, min(32, os.cpu_count() or 1))
_POOL = ThreadPoolExecutor(_NT) if _NT > 1 else None


def _chunked(fn, x, *rest):
    """fn applied to row chunks of x (and same-shaped arrays in rest); results concatenated."""
    if _POOL is None or x.ndim == 0 or x.shape[0] < 2 * _NT or x.size < (1 << 16):
        return fn(x, *rest)
    edges = np.linspace(0, x.shape[0], _NT + 1).astype(int)
    parts = list(_POOL.map(lambda k: fn(x[edges[k]:edges[k + 1]], *(r[edges[k]:edges[k + 1]] for r in rest)),
                           range(_NT)))
    return np.concatenate(parts, axis=0)


# ------------------------------------------------------------------ counter-based RNG
def splitmix64(x):
    """Vectorised splitmix64 over uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _sm_int(x: int) -> int:
    return int(splitmix64(np.uint64(x & M64)))


def synthetic_tokens(seq: int, seqs: int, vocab: int, data_seed: int, first: int, count: int,
                     causal: bool = True, pad_token: int = 0):
    """amdp_synthetic_tokens: arithmetic-progression token streams with 1/8 noise; causal ->
    next-token labels; otherwise BERT MLM (15% positions, 80/10/10 [MASK]/random/keep,
    [MASK] = vocab - 1, label -1 elsewhere).  pad_token > 0 (bidirectional only): each sequence
    keeps a length in [S/2, S] drawn from bits 40.. of its seed word; real tokens equal to the
    pad id become (pad + 1) % V, positions past the length hold the pad id with label -1."""
    T = seq * seqs
    inputs = np.empty((count, T), np.int32)
    labels = np.empty((count, T), np.int32)
    p = np.arange(seq + 1, dtype=np.uint64)
    for j in range(count):
        mb = first + j
        for b in range(seqs):
            r = _sm_int((data_seed * 0x100000001B3 + mb * 1024 + b) & M64)
            start, stride = r % vocab, 1 + (r >> 32) % 7
            with np.errstate(over="ignore"):
                nz = splitmix64(np.uint64(r) + p + np.uint64(1))
            noisy = (nz & np.uint64(7)) == 0
            prog = (np.uint64(start) + p * np.uint64(stride)) % np.uint64(vocab)
            tok = np.where(noisy, (nz >> np.uint64(8)) % np.uint64(vocab), prog).astype(np.int64)
            sl = slice(b * seq, (b + 1) * seq)
            if causal:
                inputs[j, sl] = tok[:seq]
                labels[j, sl] = tok[1:]
            else:
                with np.errstate(over="ignore"):
                    hm = splitmix64(np.uint64(r ^ 0xA5A5A5A5A5A5A5A5) + p[:seq])
                masked = (hm % np.uint64(100)) < 15
                act = (hm >> np.uint64(8)) % np.uint64(10)
                rnd = ((hm >> np.uint64(16)) % np.uint64(vocab)).astype(np.int64)
                inp = np.where(masked & (act < 8), vocab - 1, np.where(masked & (act == 8), rnd, tok[:seq]))
                lab = np.where(masked, tok[:seq], -1)
                if pad_token > 0:
                    n = seq // 2 + (r >> 40) % (seq - seq // 2 + 1)
                    inp = np.where(inp == pad_token, (pad_token + 1) % vocab, inp)
                    inp[n:] = pad_token
                    lab[n:] = -1
                inputs[j, sl] = inp
                labels[j, sl] = lab
    return inputs, labels


def normal_init(n: int, seed: int, std: float) -> np.ndarray:
    """amdp_fill_normal_bf16_f32: Box-Muller on splitmix64(key + 2i), (key + 2i + 1), fp64 -> fp32."""
    key = np.uint64(_sm_int(seed))
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        r1 = splitmix64(key + np.uint64(2) * i)
        r2 = splitmix64(key + np.uint64(2) * i + np.uint64(1))
    u1 = ((r1 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (r2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)
    return (float(np.float32(std)) * z).astype(np.float32)


def _bf16(x):
    a = np.array(x, np.float32, copy=True, order="C")
    u = a.view(np.uint32)
    r = (u >> np.uint32(16)) & np.uint32(1)
    r += np.uint32(0x7FFF)
    u += r
    u &= np.uint32(0xFFFF0000)
    return a


def bf16(x):
    """Round-to-nearest-even to bf16, returned as float32 values (uint32 arithmetic on a
    float32 copy; NaN payloads are not preserved)."""
    x = np.asarray(x)
    return _chunked(_bf16, x) if x.ndim >= 1 else _bf16(x)


# ------------------------------------------------------------------ model
@dataclass
class Model:
    layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    seq: int
    seqs: int = 4
    causal: bool = True
    seed: int = 1234
    pad_token: int = 0  # > 0 (bidirectional): keys at/after a sequence's first pad id are masked
    ln_eps: float = 1e-5
    std: float = 0.02

    @property
    def T(self):
        return self.seq * self.seqs


def stage_param_specs(m: Model, stage: int, depth: int, l0: int, l1: int):
    """(name, rows, cols, global_index, init, std) in the engine's flat order (gpt_stage.cu)."""
    std = np.float32(m.std)
    proj = np.float32(np.float32(m.std) / np.sqrt(np.float32(2.0 * m.layers)))
    out = []
    if stage == 0:
        out += [("wte", m.vocab, m.hidden, 0, 0, std), ("wpe", m.seq, m.hidden, 1, 0, std)]
    for l in range(l0, l1):
        g, p = 16 + 8 * l, f"layer{l}."
        out += [(p + "ln1.gamma", 1, m.hidden, g, 1, 0), (p + "ln1.beta", 1, m.hidden, g + 1, 2, 0),
                (p + "attn.qkv", 3 * m.hidden, m.hidden, g + 2, 0, std),
                (p + "attn.out", m.hidden, m.hidden, g + 3, 0, proj),
                (p + "ln2.gamma", 1, m.hidden, g + 4, 1, 0), (p + "ln2.beta", 1, m.hidden, g + 5, 2, 0),
                (p + "mlp.fc1", m.ffn, m.hidden, g + 6, 0, std),
                (p + "mlp.fc2", m.hidden, m.ffn, g + 7, 0, proj)]
    if stage == depth - 1:
        out += [("lnf.gamma", 1, m.hidden, 2, 1, 0), ("lnf.beta", 1, m.hidden, 3, 2, 0),
                ("head", m.vocab, m.hidden, 4, 0, std)]
    return out


def init_stage(m: Model, specs) -> Dict[str, np.ndarray]:
    P = {}
    for name, r, c, gidx, init, sd in specs:
        if init == 0:
            P[name] = normal_init(r * c, (m.seed * 1000003 + gidx) & M64, float(sd)).reshape(r, c)
        else:
            P[name] = np.full((r, c), 1.0 if init == 1 else 0.0, np.float32)
        if r == 1:
            P[name] = P[name].reshape(c)
    return P


def _gelu1(x):
    x2 = x * x
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * x * (1.0 + 0.044715 * x2)))


def _gelu_grad1(x):
    x2 = x * x
    t = np.tanh(0.7978845608028654 * x * (1.0 + 0.044715 * x2))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x2)


def _gelu(x):
    return _chunked(_gelu1, x)


def _gelu_grad(x):
    return _chunked(_gelu_grad1, x)


class StageMath:
    """Forward/backward of one stage in fp64, rounding to bf16 where the GPU stores bf16."""

    def __init__(self, m: Model, stage: int, depth: int, l0: int, l1: int, emulate_bf16: bool = True):
        self.m, self.stage, self.depth, self.l0, self.l1 = m, stage, depth, l0, l1
        self.rb = (lambda x: bf16(x).astype(np.float64)) if emulate_bf16 else (lambda x: np.asarray(x, np.float64))

    def _ln(self, x, g, b):
        mu = x.mean(-1, keepdims=True)
        var = ((x - mu) ** 2).mean(-1, keepdims=True)
        rstd = 1.0 / np.sqrt(var + self.m.ln_eps)
        return (x - mu) * rstd * g + b, mu, rstd

    def _ln_bwd(self, dy, x, g, mu, rstd):
        xh = (x - mu) * rstd
        dxh = dy * g
        dx = rstd * (dxh - dxh.mean(-1, keepdims=True) - xh * (dxh * xh).mean(-1, keepdims=True))
        return dx, (dy * xh).sum(0), dy.sum(0)

    def _lens(self, tokens):
        """Valid key length per sequence: the first pad position (executor.cu run(), >= 1)."""
        m = self.m
        if m.pad_token <= 0 or m.causal:
            return [m.seq] * m.seqs
        out = []
        for sq in np.asarray(tokens).reshape(m.seqs, m.seq):
            hit = np.nonzero(sq == m.pad_token)[0]
            out.append(max(1, int(hit[0])) if hit.size else m.seq)
        return out

    def _attn_seq(self, qkv, klen=None):
        """One sequence: qkv [S, 3hd] -> (o [S, h], p [H, S, S]); keys >= klen masked."""
        m = self.m
        S, H, D = m.seq, m.heads, m.hidden // m.heads
        q, k, v = qkv.reshape(S, 3, H, D).transpose(1, 2, 0, 3)
        s = q @ k.transpose(0, 2, 1) / math.sqrt(D)
        if m.causal:
            s = np.where(np.triu(np.ones((S, S), bool), 1), -np.inf, s)
        if klen is not None and klen < S:
            s[:, :, klen:] = -np.inf
        s = s - s.max(-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(-1, keepdims=True)
        return (p @ v).transpose(1, 0, 2).reshape(S, H * D), p

    def _attn(self, qkv, lens=None):
        m = self.m
        seqs = qkv.reshape(m.seqs, m.seq, -1)
        lens = lens if lens is not None else [None] * m.seqs
        res = list(_POOL.map(self._attn_seq, seqs, lens)) if _POOL else \
            [self._attn_seq(x, n) for x, n in zip(seqs, lens)]
        return np.concatenate([r[0] for r in res], 0), np.stack([r[1] for r in res], 0)

    def _attn_bwd_seq(self, qkv, p, do):
        m = self.m
        S, H, D = m.seq, m.heads, m.hidden // m.heads
        q, k, v = qkv.reshape(S, 3, H, D).transpose(1, 2, 0, 3)
        dO = do.reshape(S, H, D).transpose(1, 0, 2)
        dv = p.transpose(0, 2, 1) @ dO
        dp = dO @ v.transpose(0, 2, 1)
        ds = p * (dp - (dp * p).sum(-1, keepdims=True)) / math.sqrt(D)
        dq, dk = ds @ k, ds.transpose(0, 2, 1) @ q
        return np.stack([dq, dk, dv], 0).transpose(2, 0, 1, 3).reshape(S, 3 * H * D)

    def _attn_bwd(self, qkv, p, do):
        m = self.m
        args = list(zip(qkv.reshape(m.seqs, m.seq, -1), p, do.reshape(m.seqs, m.seq, -1)))
        res = list(_POOL.map(lambda a: self._attn_bwd_seq(*a), args)) if _POOL else \
            [self._attn_bwd_seq(*a) for a in args]
        return np.concatenate(res, 0)

    def forward(self, W, x_in, tokens, labels):
        rb, m = self.rb, self.m
        cache = {"x_in": x_in, "lens": self._lens(tokens)}
        if self.stage == 0:
            x = rb(W["wte"][tokens] + W["wpe"][np.arange(m.T) % m.seq])
            cache["x0"] = x
        else:
            x = x_in
        cache["layers"] = []
        for l in range(self.l0, self.l1):
            p = f"layer{l}."
            c = {"x": x}
            a, c["mu1"], c["r1"] = self._ln(x, W[p + "ln1.gamma"], W[p + "ln1.beta"])
            c["ln1"] = a = rb(a)
            c["qkv"] = qkv = rb(a @ W[p + "attn.qkv"].T)
            o, c["p"] = self._attn(qkv, cache["lens"])
            c["o"] = o = rb(o)
            c["hmid"] = hm = rb(x + o @ W[p + "attn.out"].T)
            a2, c["mu2"], c["r2"] = self._ln(hm, W[p + "ln2.gamma"], W[p + "ln2.beta"])
            c["ln2"] = a2 = rb(a2)
            u = a2 @ W[p + "mlp.fc1"].T
            c["u"] = rb(u)
            c["f"] = rb(_gelu(c["u"]))  # of the stored (bf16) pre-activation, as the fc1 epilogue
            x = rb(hm + c["f"] @ W[p + "mlp.fc2"].T)
            cache["layers"].append(c)
        loss = None
        if self.stage == self.depth - 1:
            cache["xf"] = x
            lf, cache["muf"], cache["rf"] = self._ln(x, W["lnf.gamma"], W["lnf.beta"])
            cache["lnf"] = lf = rb(lf)
            logits = rb(lf @ W["head"].T)
            mx = logits.max(-1, keepdims=True)
            lse = (mx + np.log(np.exp(logits - mx).sum(-1, keepdims=True)))[:, 0]
            valid = labels >= 0
            cnt = max(1, int(valid.sum()))  # mean over labelled tokens (all for GPT)
            rows = np.arange(m.T)[valid]
            loss = float((lse[valid] - logits[rows, labels[valid]]).sum() / cnt)
            prob = np.exp(logits - lse[:, None])
            prob[rows, labels[valid]] -= 1.0
            prob[~valid] = 0.0
            cache["dlogits"] = rb(prob / cnt)
            return None, cache, loss
        return x, cache, loss

    def backward(self, W, cache, g_in, tokens, grads):
        rb, m = self.rb, self.m
        if self.stage == self.depth - 1:
            dl = cache["dlogits"]
            dlnf = rb(dl @ W["head"])
            grads["head"] += dl.T @ cache["lnf"]
            g, dg, db = self._ln_bwd(dlnf, cache["xf"], W["lnf.gamma"], cache["muf"], cache["rf"])
            grads["lnf.gamma"] += dg
            grads["lnf.beta"] += db
            g = rb(g)
        else:
            g = g_in
        for li in reversed(range(self.l1 - self.l0)):
            l = self.l0 + li
            p, c = f"layer{l}.", cache["layers"][li]
            dU = rb((g @ W[p + "mlp.fc2"]) * _gelu_grad(c["u"]))
            grads[p + "mlp.fc2"] += g.T @ c["f"]
            dln2 = rb(dU @ W[p + "mlp.fc1"])
            grads[p + "mlp.fc1"] += dU.T @ c["ln2"]
            dx, dg, db = self._ln_bwd(dln2, c["hmid"], W[p + "ln2.gamma"], c["mu2"], c["r2"])
            grads[p + "ln2.gamma"] += dg
            grads[p + "ln2.beta"] += db
            dh = rb(g + dx)
            dO = rb(dh @ W[p + "attn.out"])
            grads[p + "attn.out"] += dh.T @ c["o"]
            dqkv = rb(self._attn_bwd(c["qkv"], c["p"], dO))
            dln1 = rb(dqkv @ W[p + "attn.qkv"])
            grads[p + "attn.qkv"] += dqkv.T @ c["ln1"]
            dx, dg, db = self._ln_bwd(dln1, c["x"], W[p + "ln1.gamma"], c["mu1"], c["r1"])
            grads[p + "ln1.gamma"] += dg
            grads[p + "ln1.beta"] += db
            g = rb(dh + dx)
        if self.stage == 0:
            np.add.at(grads["wte"], tokens, g)
            grads["wpe"] += g.reshape(m.seqs, m.seq, -1).sum(0)
            return None
        return g


# ------------------------------------------------------------------ optimizer (optim.hpp:234-268)
@dataclass
class Opt:
    kind: str = "adamw"      # sgd | momentum | adamtype (reference rule) | adamw
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0
    clamp_min: float = 1e-8
    clamp_max: float = 1e6


def apply_update(opt: Opt, theta, m, v, g, step: int):
    """In place; restates detail::apply_update (no clip) plus the AdamW mode."""
    if opt.kind == "sgd":
        theta -= opt.lr * g
    elif opt.kind == "momentum":
        m[...] = opt.beta1 * m + (1 - opt.beta1) * g
        theta -= opt.lr * m
    elif opt.kind == "adamtype":
        m[...] = opt.beta1 * m + (1 - opt.beta1) * g
        v[...] = opt.beta2 * v + (1 - opt.beta2) * g * g
        pre = np.clip(1.0 / (np.sqrt(v) + opt.eps), opt.clamp_min, opt.clamp_max)
        theta -= opt.lr * pre * m
    else:
        m[...] = opt.beta1 * m + (1 - opt.beta1) * g
        v[...] = opt.beta2 * v + (1 - opt.beta2) * g * g
        mh, vh = m / (1 - opt.beta1 ** step), v / (1 - opt.beta2 ** step)
        theta -= opt.lr * (mh / (np.sqrt(vh) + opt.eps) + opt.weight_decay * theta)


# ------------------------------------------------------------------ trace replay
def parse_timeline_csv(text: str):
    rows = list(csv.DictReader(io.StringIO(text)))
    from fractions import Fraction
    ev = []
    for idx, r in enumerate(rows):
        s, d = Fraction(r["start"]), Fraction(r["duration"])
        ev.append(dict(device=int(r["device"]), kind=r["kind"], stage=int(r["stage"]),
                       minibatch=int(r["minibatch"]), pipeline=int(r["pipeline"]),
                       window=int(r["window"]), preloaded=int(r["preloaded"]), start=s, dur=d, row=idx))
    return ev


def replay(trace_csv: str, m: Model, partition: List[int], opt: Opt, threshold: int,
           inputs: np.ndarray, labels: np.ndarray, emulate_bf16: bool = True,
           update_div: Optional[int] = None):
    """Executes the reference trace on the CPU.  Returns (losses[M], params per stage (fp32
    master dicts), version trace rows {(kind, stage, minibatch): version}).

    Window events (builder.hpp:260-338): Broadcast(w, i) (ZeRO) rewrites every replica of
    stage i; Update(w, i, p) advances replica p only (analysis.hpp:47-52: a Forward / Backward
    of pipeline p counts the Broadcasts of its stage and the Updates of its own pipeline).
    Replicas apply the same all-reduced gradient, so the first Update of (stage, window) takes
    the optimizer step and the others switch to its result.  The optimizer step number is the
    event's minibatch field + 1 (window w, or minibatch j for PipeDreamAsync's per-backward
    Update); the gradient is divided by `update_div` (default: the threshold; 1 for
    PipeDreamAsync)."""
    ev = parse_timeline_csv(trace_csv)
    # zero-duration window events complete at their start: apply before compute starting then
    ev.sort(key=lambda e: (e["start"], e["dur"] > 0, e["device"], e["row"]))
    div = threshold if update_div is None else update_div
    depth = len(partition)
    npipe = 1 + max(e["pipeline"] for e in ev)
    bounds = np.concatenate([[0], np.cumsum(partition)]).astype(int)
    specs = [stage_param_specs(m, i, depth, bounds[i], bounds[i + 1]) for i in range(depth)]
    master = [{k: v.astype(np.float64) for k, v in init_stage(m, s).items()} for s in specs]
    mom = [{k: np.zeros_like(v) for k, v in st.items()} for st in master]
    vel = [{k: np.zeros_like(v) for k, v in st.items()} for st in master]
    grads = [{k: np.zeros_like(v) for k, v in st.items()} for st in master]
    math_ = [StageMath(m, i, depth, bounds[i], bounds[i + 1], emulate_bf16) for i in range(depth)]
    rb = (lambda x: bf16(x).astype(np.float64)) if emulate_bf16 else (lambda x: x)

    def working(st):  # the bf16 working copy the kernels read
        return {k: rb(v.astype(np.float32)) if v.ndim == 2 else v.astype(np.float32).astype(np.float64)
                for k, v in st.items()}

    works = [[working(st)] for st in master]  # works[i][k]: stage i after k optimizer steps
    ver = {(i, p): 0 for i in range(depth) for p in range(npipe)}  # replica -> steps it reads
    stepped = set()
    acts, caches, gsend = {}, {}, {}
    M = inputs.shape[0]
    losses = np.zeros(M)
    seen = {}
    for e in ev:
        i, j, p = e["stage"], e["minibatch"], e["pipeline"]
        if e["kind"] == "Forward":
            seen[("Forward", i, j)] = ver[(i, p)]
            out, cache, loss = math_[i].forward(works[i][ver[(i, p)]], acts.get((i, j)), inputs[j], labels[j])
            caches[(i, j)] = cache
            if out is not None:
                acts[(i + 1, j)] = out
            if loss is not None:
                losses[j] = loss
        elif e["kind"] == "Backward":
            seen[("Backward", i, j)] = ver[(i, p)]
            g = math_[i].backward(works[i][ver[(i, p)]], caches.pop((i, j)), gsend.pop((i, j), None),
                                  inputs[j], grads[i])
            if g is not None:
                gsend[(i - 1, j)] = g
        elif e["kind"] in ("Broadcast", "Update"):
            if (i, j) not in stepped:  # first window event of (stage, window / minibatch)
                stepped.add((i, j))
                for k in master[i]:
                    apply_update(opt, master[i][k], mom[i][k], vel[i][k], grads[i][k] / div, j + 1)
                    grads[i][k][...] = 0
                works[i].append(working(master[i]))
            for q in (range(npipe) if e["kind"] == "Broadcast" else (p,)):
                ver[(i, q)] = len(works[i]) - 1
    return losses, master, seen


def flat_stage(master_stage: Dict[str, np.ndarray], layout: List[dict], numel: int) -> np.ndarray:
    """Packs a stage's parameters into the engine's flat layout (engine.plan()['stages'][i])."""
    out = np.zeros(numel, np.float64)
    for p in layout:
        out[p["offset"]:p["offset"] + p["rows"] * p["cols"]] = master_stage[p["name"]].reshape(-1)
    return out
