"""Python mirror of the reference's ppsim API, backed by libamdp.so (include/amdp_sched.h).

Same names and meaning as /root/reference/proj/include/ppsim: ClusterSpec/PolicyConfig
(types.hpp:60-119), build (builder.hpp:145), simulate (engine.hpp:28), bubble_ratio
(engine.hpp:166), mismatch_report / window_mismatch / memory_report (analysis.hpp),
validate_* (validate.hpp), timeline_csv (serialize.hpp:41).  Errors map to the reference's
exception types: ValueError for std::invalid_argument, RuntimeError for
std::runtime_error ("dependency cycle: ...", "deadlock: ..."), OverflowError /
ZeroDivisionError for Rat arithmetic.  Exact times are fractions.Fraction.
"""
from __future__ import annotations

import ctypes
import enum
import json
from ctypes import POINTER, Structure, byref, c_char_p, c_int, c_int64, c_size_t, c_void_p
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

from ._native import lib

Rat = Fraction


class Kind(enum.IntEnum):
    Forward = 0
    Backward = 1
    Reduce = 2
    Broadcast = 3
    Update = 4


class Policy(enum.IntEnum):
    AMDP = 0
    DAPPLE = 1
    GPipe = 2
    Interleaved1F1B = 3
    Chimera = 4
    PipeDreamAsync = 5


def kind_rank(k: Kind) -> int:
    return int(k)


def policy_from_name(s: str) -> Optional[Policy]:
    return Policy.__members__.get(s)


# ------------------------------------------------------------------ C structs
class _Rat(Structure):
    _fields_ = [("num", c_int64), ("den", c_int64)]


class _Cluster(Structure):
    _fields_ = [("depth", c_int), ("devices", c_int),
                ("fwd_cost", POINTER(_Rat)), ("n_fwd", c_int),
                ("bwd_cost", POINTER(_Rat)), ("n_bwd", c_int),
                ("update_cost", _Rat), ("comm_cost", _Rat),
                ("num_nodes", c_int), ("node_sizes", POINTER(c_int)),
                ("node_devices", POINTER(c_int)),
                ("has_inter_node_cost", c_int), ("inter_node_cost", _Rat)]


class _Policy(Structure):
    _fields_ = [("policy", c_int), ("injection_limit", c_int), ("num_pipelines", c_int),
                ("accumulation_threshold", c_int), ("num_minibatches", c_int),
                ("zero_enabled", c_int), ("injection_override", c_int)]


class _TaskInfo(Structure):
    _fields_ = [("kind", c_int), ("stage", c_int), ("minibatch", c_int), ("pipeline", c_int),
                ("device", c_int), ("window", c_int), ("preloaded", c_int), ("duration", _Rat)]


class _Event(Structure):
    _fields_ = [("kind", c_int), ("stage", c_int), ("minibatch", c_int), ("pipeline", c_int),
                ("device", c_int), ("window", c_int), ("preloaded", c_int),
                ("start", _Rat), ("duration", _Rat)]


_ERRBUF = 4096
_H = c_void_p


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype, f.argtypes = res, args


_sig("amdp_validate", c_int, [POINTER(_Policy), POINTER(_Cluster), c_char_p, c_size_t])
_sig("amdp_validate_cluster", c_int, [POINTER(_Cluster), c_char_p, c_size_t])
_sig("amdp_validate_policy", c_int, [POINTER(_Policy), POINTER(_Cluster), c_char_p, c_size_t])
_sig("amdp_schedule_clone", c_void_p, [c_void_p])
_sig("amdp_map_stage_to_device", c_int, [c_int, c_int, c_int, POINTER(c_int), c_char_p, c_size_t])
_sig("amdp_default_num_pipelines", c_int, [c_int, POINTER(c_int), c_char_p, c_size_t])
_sig("amdp_preload_count", c_int, [_Rat, _Rat, POINTER(c_int), c_char_p, c_size_t])
_sig("amdp_schedule_build", _H, [POINTER(_Policy), POINTER(_Cluster), c_char_p, c_size_t])
_sig("amdp_graph_new", _H, [c_int, c_int, c_int, c_int, POINTER(_Cluster)])
_sig("amdp_graph_add_task", c_int, [_H, POINTER(_TaskInfo)])
_sig("amdp_graph_add_dep", c_int, [_H, c_int, c_int])
_sig("amdp_graph_add_lane", c_int, [_H, POINTER(c_int), c_int])
_sig("amdp_timeline_new", _H, [c_int, c_int, c_int, c_int, POINTER(_Event), c_int, POINTER(_Cluster)])
_sig("amdp_schedule_free", None, [_H])
_sig("amdp_schedule_simulate", c_int, [_H, c_char_p, c_size_t])
_sig("amdp_schedule_num_tasks", c_int, [_H])
_sig("amdp_schedule_tasks", c_int, [_H, POINTER(_TaskInfo), c_int])
_sig("amdp_schedule_num_deps", c_int, [_H])
_sig("amdp_schedule_deps", c_int, [_H, POINTER(c_int), c_int])
_sig("amdp_schedule_order", c_int, [_H, POINTER(c_int), c_int])
_sig("amdp_schedule_num_events", c_int, [_H])
_sig("amdp_schedule_events", c_int, [_H, POINTER(_Event), c_int])
_sig("amdp_schedule_makespan", c_int, [_H, POINTER(_Rat)])
_sig("amdp_schedule_bubble", c_int, [_H, c_int, POINTER(_Rat), c_char_p, c_size_t])
_sig("amdp_schedule_text", c_size_t, [_H, c_int, c_char_p, c_size_t])
_sig("amdp_schedule_report_json", c_size_t, [_H, POINTER(_Policy), c_int, c_char_p, c_size_t])

_EINVAL, _ERUNTIME, _EARITH, _ESTATE = -1, -2, -3, -4


def _raise(rc: int, err: ctypes.Array) -> None:
    if rc == 0:
        return
    msg = err.value.decode()
    if rc == _EINVAL:
        raise ValueError(msg)
    if rc == _EARITH:
        if "zero" in msg or "division" in msg:
            raise ZeroDivisionError(msg)
        raise OverflowError(msg)
    if rc == _ESTATE:
        raise RuntimeError("invalid handle state")
    raise RuntimeError(msg)


def _r(x) -> _Rat:
    f = Fraction(x)
    return _Rat(f.numerator, f.denominator)


def _f(r: _Rat) -> Fraction:
    return Fraction(r.num, r.den)


# ------------------------------------------------------------------ config types
@dataclass
class ClusterSpec:
    depth: int = 0
    devices: int = 0
    fwd_cost: List[Fraction] = field(default_factory=list)
    bwd_cost: List[Fraction] = field(default_factory=list)
    update_cost: Fraction = Fraction(0)
    comm_cost: Fraction = Fraction(0)
    nodes: List[List[int]] = field(default_factory=list)
    inter_node_cost: Optional[Fraction] = None

    @staticmethod
    def uniform(depth, devices, fwd, bwd, update=0, comm=0) -> "ClusterSpec":
        return ClusterSpec(depth, devices, [Fraction(fwd)] * depth, [Fraction(bwd)] * depth,
                           Fraction(update), Fraction(comm))

    def mean_fwd(self) -> Fraction:
        return sum(map(Fraction, self.fwd_cost), Fraction(0)) / len(self.fwd_cost)

    def mean_bwd(self) -> Fraction:
        return sum(map(Fraction, self.bwd_cost), Fraction(0)) / len(self.bwd_cost)

    def node_of(self, device: int) -> int:
        for g, grp in enumerate(self.nodes):
            if device in grp:
                return g
        return 0

    def gap(self, a: int, b: int) -> Fraction:
        if a == b:
            return Fraction(0)
        if self.nodes and self.inter_node_cost is not None and self.node_of(a) != self.node_of(b):
            return Fraction(self.inter_node_cost)
        return Fraction(self.comm_cost)

    def _c(self):
        fw = (_Rat * max(1, len(self.fwd_cost)))(*[_r(x) for x in self.fwd_cost])
        bw = (_Rat * max(1, len(self.bwd_cost)))(*[_r(x) for x in self.bwd_cost])
        sizes = (c_int * max(1, len(self.nodes)))(*[len(g) for g in self.nodes])
        members = [d for g in self.nodes for d in g]
        devs = (c_int * max(1, len(members)))(*members)
        c = _Cluster(self.depth, self.devices, fw, len(self.fwd_cost), bw, len(self.bwd_cost),
                     _r(self.update_cost), _r(self.comm_cost), len(self.nodes), sizes, devs,
                     int(self.inter_node_cost is not None),
                     _r(self.inter_node_cost if self.inter_node_cost is not None else 0))
        c._keep = (fw, bw, sizes, devs)
        return c


@dataclass
class PolicyConfig:
    policy: Policy = Policy.DAPPLE
    injection_limit: int = 1
    num_pipelines: int = 1
    accumulation_threshold: int = 1
    num_minibatches: int = 1
    zero_enabled: bool = False
    injection_override: bool = False

    def _c(self):
        return _Policy(int(self.policy), self.injection_limit, self.num_pipelines,
                       self.accumulation_threshold, self.num_minibatches, int(self.zero_enabled),
                       int(self.injection_override))


@dataclass
class Task:
    kind: Kind = Kind.Forward
    stage: int = 0
    minibatch: int = 0
    pipeline: int = 0
    device: int = 0
    duration: Fraction = Fraction(0)
    window: int = 0
    preloaded: bool = False


@dataclass
class TaskEvent:
    kind: Kind = Kind.Forward
    stage: int = 0
    minibatch: int = 0
    pipeline: int = 0
    device: int = 0
    start: Fraction = Fraction(0)
    duration: Fraction = Fraction(0)
    preloaded: bool = False
    window: int = 0

    def finish(self) -> Fraction:
        return self.start + self.duration


class _Handle:
    def __init__(self, h):
        if not h:
            raise RuntimeError("null schedule handle")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib.amdp_schedule_free(self.h)
            self.h = None


class TaskGraph:
    """builder.hpp:28-37.  Either produced by build() (handle-backed) or assembled by hand."""

    def __init__(self, policy=Policy.DAPPLE, depth=0, devices=0, threshold=1):
        self.policy, self.depth, self.devices, self.threshold = policy, depth, devices, threshold
        self.tasks: List[Task] = []
        self.deps: List[Tuple[int, int]] = []
        self.lanes: List[List[int]] = []
        self._built: Optional[_Handle] = None
        self._built_cluster: Optional[ClusterSpec] = None

    @classmethod
    def _from_handle(cls, h: _Handle, cfg: PolicyConfig, cl: ClusterSpec) -> "TaskGraph":
        g = cls(cfg.policy, cl.depth, cl.devices, cfg.accumulation_threshold)
        n = lib.amdp_schedule_num_tasks(h.h)
        arr = (_TaskInfo * max(1, n))()
        lib.amdp_schedule_tasks(h.h, arr, n)
        g.tasks = [Task(Kind(t.kind), t.stage, t.minibatch, t.pipeline, t.device, _f(t.duration),
                        t.window, bool(t.preloaded)) for t in arr[:n]]
        nd = lib.amdp_schedule_num_deps(h.h)
        dd = (c_int * max(2, 2 * nd))()
        lib.amdp_schedule_deps(h.h, dd, nd)
        g.deps = [(dd[2 * i], dd[2 * i + 1]) for i in range(nd)]
        g._built, g._built_cluster = h, cl
        return g

    def _handle_for(self, cl: ClusterSpec) -> _Handle:
        h = _Handle(lib.amdp_graph_new(int(self.policy), self.depth, self.devices, self.threshold,
                                       byref(cl._c())))
        for t in self.tasks:
            ti = _TaskInfo(int(t.kind), t.stage, t.minibatch, t.pipeline, t.device, t.window,
                           int(t.preloaded), _r(t.duration))
            lib.amdp_graph_add_task(h.h, byref(ti))
        for a, b in self.deps:
            lib.amdp_graph_add_dep(h.h, a, b)
        for lane in self.lanes:
            arr = (c_int * max(1, len(lane)))(*lane)
            lib.amdp_graph_add_lane(h.h, arr, len(lane))
        return h


class Timeline:
    """types.hpp:135-150; handle-backed so analyses run in the native library."""

    def __init__(self, h: _Handle, policy: Policy, depth: int, devices: int, threshold: int,
                 cluster: ClusterSpec, order: Optional[List[int]] = None):
        self._h, self.policy, self.depth, self.devices, self.threshold = h, policy, depth, devices, threshold
        self._cluster = cluster
        self.order = order
        n = lib.amdp_schedule_num_events(h.h)
        arr = (_Event * max(1, n))()
        lib.amdp_schedule_events(h.h, arr, n)
        self.per_device: List[List[TaskEvent]] = [[] for _ in range(devices)]
        for e in arr[:n]:
            self.per_device[e.device].append(
                TaskEvent(Kind(e.kind), e.stage, e.minibatch, e.pipeline, e.device, _f(e.start),
                          _f(e.duration), bool(e.preloaded), e.window))
        ms = _Rat()
        lib.amdp_schedule_makespan(h.h, byref(ms))
        self.makespan = _f(ms)

    @staticmethod
    def from_events(events: Sequence[TaskEvent], policy: Policy, depth: int, devices: int,
                    threshold: int = 1, cluster: Optional[ClusterSpec] = None) -> "Timeline":
        cl = cluster or ClusterSpec(depth, devices)
        arr = (_Event * max(1, len(events)))(*[
            _Event(int(e.kind), e.stage, e.minibatch, e.pipeline, e.device, e.window,
                   int(e.preloaded), _r(e.start), _r(e.duration)) for e in events])
        h = _Handle(lib.amdp_timeline_new(int(policy), depth, devices, threshold, arr, len(events),
                                          byref(cl._c())))
        return Timeline(h, policy, depth, devices, threshold, cl)

    def flat(self) -> List[TaskEvent]:
        return [e for dev in self.per_device for e in dev]

    def report(self, cfg: Optional[PolicyConfig] = None, warmup: int = 0) -> dict:
        pc = byref(cfg._c()) if cfg is not None else None
        n = lib.amdp_schedule_report_json(self._h.h, pc, warmup, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib.amdp_schedule_report_json(self._h.h, pc, warmup, buf, n + 1)
        return json.loads(buf.value.decode())

    def _text(self, which: int) -> str:
        n = lib.amdp_schedule_text(self._h.h, which, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib.amdp_schedule_text(self._h.h, which, buf, n + 1)
        return buf.raw[:n].decode()


# ------------------------------------------------------------------ functions
def _msgs(n: int, buf) -> List[str]:
    return buf.value.decode().split("\n") if n else []


def validate_cluster(c: ClusterSpec) -> List[str]:
    buf = ctypes.create_string_buffer(1 << 16)
    return _msgs(lib.amdp_validate_cluster(byref(c._c()), buf, len(buf)), buf)


def validate_policy(p: PolicyConfig, c: ClusterSpec) -> List[str]:
    buf = ctypes.create_string_buffer(1 << 16)
    return _msgs(lib.amdp_validate_policy(byref(p._c()), byref(c._c()), buf, len(buf)), buf)


def validate_causality(t: Timeline, c: ClusterSpec) -> List[str]:
    t2 = Timeline.from_events(t.flat(), t.policy, t.depth, t.devices, t.threshold, c)
    return t2.report()["causality_issues"]


def validate_non_overlap(t: Timeline) -> List[str]:
    return t.report()["overlap_issues"]


def map_stage_to_device(pipeline: int, stage: int, depth: int) -> int:
    out, err = c_int(), ctypes.create_string_buffer(_ERRBUF)
    _raise(lib.amdp_map_stage_to_device(pipeline, stage, depth, byref(out), err, _ERRBUF), err)
    return out.value


def default_num_pipelines(depth: int) -> int:
    out, err = c_int(), ctypes.create_string_buffer(_ERRBUF)
    _raise(lib.amdp_default_num_pipelines(depth, byref(out), err, _ERRBUF), err)
    return out.value


def preload_count(bwd, fwd) -> int:
    out, err = c_int(), ctypes.create_string_buffer(_ERRBUF)
    _raise(lib.amdp_preload_count(_r(bwd), _r(fwd), byref(out), err, _ERRBUF), err)
    return out.value


def active_ratio(injection_limit: int, depth: int) -> Fraction:
    return Fraction(injection_limit, depth)


def build(cfg: PolicyConfig, cl: ClusterSpec) -> TaskGraph:
    err = ctypes.create_string_buffer(_ERRBUF)
    h = lib.amdp_schedule_build(byref(cfg._c()), byref(cl._c()), err, _ERRBUF)
    if not h:
        raise ValueError(err.value.decode())
    return TaskGraph._from_handle(_Handle(h), cfg, cl)


def simulate(g: TaskGraph, cl: ClusterSpec) -> Timeline:
    if g._built is not None and g._built_cluster == cl and _same_as_built(g):
        h = _Handle(lib.amdp_schedule_clone(g._built.h))
    else:
        h = g._handle_for(cl)
    err = ctypes.create_string_buffer(_ERRBUF)
    _raise(lib.amdp_schedule_simulate(h.h, err, _ERRBUF), err)
    n = lib.amdp_schedule_num_tasks(h.h)
    arr = (c_int * max(1, n))()
    lib.amdp_schedule_order(h.h, arr, n)
    return Timeline(h, g.policy, g.depth, g.devices, g.threshold, cl, list(arr[:n]))


def _same_as_built(g: TaskGraph) -> bool:
    return (not g.lanes and lib.amdp_schedule_num_tasks(g._built.h) == len(g.tasks)
            and lib.amdp_schedule_num_deps(g._built.h) == len(g.deps))


def bubble_ratio(tl: Timeline, warmup_windows: int = 0) -> Fraction:
    out, err = _Rat(), ctypes.create_string_buffer(_ERRBUF)
    _raise(lib.amdp_schedule_bubble(tl._h.h, warmup_windows, byref(out), err, _ERRBUF), err)
    return _f(out)


@dataclass
class MismatchReport:
    entries: Dict[Tuple[int, int], int]
    max_per_stage: Dict[int, int]
    missing: List[Tuple[int, int]]

    def max_overall(self) -> int:
        return max(self.entries.values(), default=0)


def mismatch_report(t: Timeline) -> MismatchReport:
    r = t.report()["mismatch"]
    return MismatchReport({(s, j): n for s, j, n in r["entries"]},
                          {s: n for s, n in r["max_per_stage"]},
                          [tuple(x) for x in r["missing"]])


@dataclass
class WindowEntry:
    window: int
    mismatched: List[int]
    window_size: int
    update_count: int


def window_mismatch(t: Timeline, depth: int) -> List[WindowEntry]:
    return [WindowEntry(w["window"], w["mismatched"], w["window_size"], w["update_count"])
            for w in t.report()["windows"]]


def memory_report(t: Timeline, policy: PolicyConfig) -> dict:
    """Unit MemoryModel (analysis.hpp:226 with MemoryModel{}); rationals as int or 'n/d'."""
    return t.report(policy)["memory"]


def reduce_broadcast_cost(replicas: int, nbytes) -> Tuple[Fraction, Fraction, Fraction]:
    if replicas < 1:
        raise ValueError("replicas must be at least 1")
    if replicas == 1:
        return Fraction(0), Fraction(0), Fraction(0)
    per = Fraction(nbytes) * Fraction(replicas - 1, replicas)
    return per, per, 2 * per


def timeline_csv(t: Timeline) -> str:
    return t._text(0)


def version_trace_csv(t: Timeline) -> str:
    return t._text(1)


def timeline_json(t: Timeline) -> dict:
    return json.loads(t._text(2))


_GANTT_COLOR = {Kind.Forward: "#3b7dd8", Kind.Backward: "#f0a030", Kind.Reduce: "#8a5cc2",
                Kind.Broadcast: "#3fae7a", Kind.Update: "#d25050"}


def gantt_svg(t: Timeline, title: str = "", window_from: Optional[int] = None,
              window_to: Optional[int] = None) -> str:
    """SVG Gantt chart of a timeline (the reference's gantt.hpp:36-100 view: one lane per
    device, one bar per task coloured by kind, preloaded forwards outlined, idle time blank),
    optionally cut to windows [window_from, window_to].  Deterministic for a given timeline;
    measured (ns) and declared (rational) timelines render alike."""
    evs = [e for e in t.flat() if (window_from is None or e.window >= window_from)
           and (window_to is None or e.window <= window_to)]
    if not evs:
        return '<svg xmlns="http://www.w3.org/2000/svg" width="10" height="10"/>\n'
    t0 = min(float(e.start) for e in evs)
    t1 = max(float(e.finish()) for e in evs)
    span = max(t1 - t0, 1e-12)
    lane, gap, x0, y0, width = 22, 4, 58, 30, 1200
    height = y0 + t.devices * (lane + gap) + 40
    sx = width / span
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{x0 + width + 12}" height="{height}" '
           f'font-family="sans-serif" font-size="11">',
           f'<rect x="0" y="0" width="{x0 + width + 12}" height="{height}" fill="white"/>',
           f'<text x="{x0}" y="16">{title or t.policy.name} - {t.depth} stages on {t.devices} devices, '
           f'span {span:.6g}</text>']
    busy = [0.0] * t.devices
    for e in sorted(evs, key=lambda e: (e.device, e.start, int(e.kind))):
        d = float(e.duration)
        if d <= 0:
            continue
        busy[e.device] += d
        x = x0 + (float(e.start) - t0) * sx
        y = y0 + e.device * (lane + gap)
        stroke = ' stroke="black" stroke-dasharray="2,2"' if e.preloaded else ""
        out.append(f'<rect x="{x:.2f}" y="{y}" width="{max(d * sx, 0.5):.2f}" height="{lane}" '
                   f'fill="{_GANTT_COLOR[e.kind]}"{stroke}><title>{e.kind.name} stage {e.stage} mb '
                   f'{e.minibatch} pipe {e.pipeline} window {e.window}</title></rect>')
    for dv in range(t.devices):
        y = y0 + dv * (lane + gap)
        out.append(f'<text x="4" y="{y + 15}">dev {dv}</text>')
        out.append(f'<text x="{x0 + width + 2}" y="{y + 15}" font-size="9">{100 * (1 - busy[dv] / span):.0f}%</text>')
    lx = x0
    for k, c in _GANTT_COLOR.items():
        out.append(f'<rect x="{lx}" y="{height - 24}" width="10" height="10" fill="{c}"/>'
                   f'<text x="{lx + 14}" y="{height - 15}">{k.name}</text>')
        lx += 95
    out.append(f'<text x="{lx + 10}" y="{height - 15}">right margin: idle share per device</text>')
    out.append("</svg>")
    return "\n".join(out) + "\n"
