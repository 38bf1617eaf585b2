"""Python mirror of the reference's scheduler interface (proj/include/batchsim),
backed by libbs_host.so through its JSON C-ABI (bs_host_call).

Names, argument meaning and error behaviour follow the reference:
  compute_schedule_dp / compute_schedule / compute_schedule_layer_units /
  compute_schedule_grouped      (dp_time.hpp:152-347)
  baseline_no_batch / baseline_batch (dp_time.hpp:358-415)
  edf_batch / tardy_dp          (deadline.hpp:42-282)
  schedule_multi / schedule_multi_shared (multi_dnn.hpp:284-301)
  segment_duration / group_layers / ProfileSet lookups (schedule.hpp:183,
  cost_model.hpp:239)
  run_sim                       (simulator.hpp:787)
std::runtime_error -> RuntimeError, std::invalid_argument -> ValueError,
std::logic_error -> LogicError.
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field
from typing import Iterable, Sequence

from ._native import host_call

INF = math.inf
kInfeasible = INF
kNoDeadline = INF


class LogicError(RuntimeError):
    pass


def f64(bits: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(bits, 16)))[0]


def bits64(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


@dataclass
class Request:
    id: int
    dnn: int = 0
    arrival: float = 0.0
    deadline: float = INF
    layer: int = 1

    def to_json(self):
        return [self.id, self.dnn, bits64(self.arrival),
                None if self.deadline == INF else bits64(self.deadline), self.layer]


def make_request(id, arrival, layer, deadline=INF, dnn=0) -> Request:
    return Request(id=id, dnn=dnn, arrival=arrival, deadline=deadline, layer=layer)


@dataclass
class Rider:
    id: int
    dnn: int
    join_layer: int
    leave_layer: int
    deposit_layer: int


@dataclass
class ScheduledSegment:
    members: list
    dnn: int
    start_layer: int
    duration: float
    finish_offset: float
    max_layer_batch: int
    riders: list = field(default_factory=list)


@dataclass
class Schedule:
    segments: list
    completion_offsets: list
    objective: float
    total_duration: float
    tardy_count: int
    drop_marks: list
    raw: dict = field(repr=False, default=None)

    def offset_of(self, rid: int) -> float:
        for i, off in self.completion_offsets:
            if i == rid:
                return off
        return INF

    @classmethod
    def from_json(cls, d: dict) -> "Schedule":
        segs = [ScheduledSegment(s["members"], s["dnn"], s["start_layer"], f64(s["duration"]),
                                 f64(s["finish_offset"]), s["max_layer_batch"],
                                 [Rider(*r) for r in s["riders"]]) for s in d["segments"]]
        return cls(segs, [(i, f64(o)) for i, o in d["completion_offsets"]], f64(d["objective"]),
                   f64(d["total_duration"]), d["tardy_count"], d["drop_marks"], d)


@dataclass
class SweepResult:
    duration: float
    max_layer_batch: int
    layer_batch: list
    start_layer: int
    feasible: bool


# ----------------------------------------------------------------- profiles

def profile_from_grids(layers: Sequence[Sequence[tuple]], max_batch: int, dnn_name="d0") -> dict:
    """Single-DNN profile; layers[k] is the (batch, ms) grid of layer k+1
    (mirrors the reference tests' profile_from_grids)."""
    return {"max_batch": max_batch,
            "components": [{"id": dnn_name + "_body",
                            "layers": [{"output_bits": 100000, "runtime_ms": [list(p) for p in g]}
                                       for g in layers]}],
            "dnns": [{"id": dnn_name, "stages": [dnn_name + "_body"]}]}


def uniform_profile(num_layers: int, grid, max_batch: int, dnn_name="d0") -> dict:
    return profile_from_grids([grid] * num_layers, max_batch, dnn_name)


def load_profile(path: str) -> str:
    return str(path)


# --------------------------------------------------------------------- calls

def _raise(err: str):
    kind, _, msg = err.partition(": ")
    if "invalid_argument" in kind:
        raise ValueError(msg)
    if "logic_error" in kind:
        raise LogicError(msg)
    raise RuntimeError(msg)


def _call(profile, fn: str, requests: Iterable[Request] = (), **kw):
    c = {"fn": fn, "requests": [r.to_json() for r in requests]}
    for k, v in kw.items():
        if v is None:
            continue
        c[k] = bits64(v) if isinstance(v, float) and k in ("now", "start_offset") else v
    out = json.loads(host_call({"job": "calls", "profile": profile, "calls": [c]}).splitlines()[0])
    if "error" in out:
        _raise(out["error"])
    return out["result"]


_GRAN = {"per_request": "request", "per_layer": "layer", "per_group": "group",
         "request": "request", "layer": "layer", "group": "group"}


def compute_schedule_dp(requests, ps, dnn, bound, granularity="per_request", groups=5,
                        extra_active=0) -> Schedule:
    return Schedule.from_json(_call(ps, "dp", requests, dnn=dnn, bound=bound,
                                    granularity=_GRAN[granularity], groups=groups,
                                    extra_active=extra_active))


def compute_schedule(requests, ps, dnn, bound) -> Schedule:
    return compute_schedule_dp(requests, ps, dnn, bound, "per_request", 0)


def compute_schedule_layer_units(requests, ps, dnn, bound) -> Schedule:
    return compute_schedule_dp(requests, ps, dnn, bound, "per_layer", 0)


def compute_schedule_grouped(requests, ps, dnn, bound, groups) -> Schedule:
    return compute_schedule_dp(requests, ps, dnn, bound, "per_group", groups)


def baseline_no_batch(requests, ps) -> Schedule:
    return Schedule.from_json(_call(ps, "no_batch", requests))


def baseline_batch(requests, ps, bound) -> Schedule:
    return Schedule.from_json(_call(ps, "batch", requests, bound=bound))


def edf_batch(requests, ps, bound, now) -> Schedule:
    return Schedule.from_json(_call(ps, "edf", requests, bound=bound, now=float(now)))


def tardy_dp(requests, ps, dnn, bound, now, granularity="per_request", groups=5,
             start_offset=0.0) -> Schedule:
    return Schedule.from_json(_call(ps, "tardy", requests, dnn=dnn, bound=bound, now=float(now),
                                    granularity=_GRAN[granularity], groups=groups,
                                    start_offset=float(start_offset)))


def schedule_multi(requests, ps, bound, granularity="per_request", groups=5, guard=6,
                   heuristic=False) -> Schedule:
    return Schedule.from_json(_call(ps, "multi", requests, bound=bound, granularity=_GRAN[granularity],
                                    groups=groups, guard=guard, heuristic=heuristic))


def schedule_multi_shared(requests, ps, bound, granularity="per_request", groups=5, guard=6,
                          heuristic=False) -> Schedule:
    return Schedule.from_json(_call(ps, "multi_shared", requests, bound=bound,
                                    granularity=_GRAN[granularity], groups=groups, guard=guard,
                                    heuristic=heuristic))


def segment_duration(layers, ps, dnn, bound) -> SweepResult:
    r = _call(ps, "segment", (), layers=list(layers), dnn=dnn, bound=bound)
    return SweepResult(f64(r["duration"]), r["max_layer_batch"], r["layer_batch"], r["start_layer"],
                       r["feasible"])


def group_layers(ps, dnn, groups) -> list[tuple[int, int]]:
    return [tuple(g) for g in _call(ps, "groups", (), dnn=dnn, groups=groups)]


def lookup_table(ps, dnn, bound) -> list[list[float]]:
    """h_k(b) for k = 1..N, b = 1..bound+1 (the last column is +inf)."""
    flat = [f64(x) for x in _call(ps, "lookup", (), dnn=dnn, bound=bound)]
    w = bound + 1
    return [flat[i:i + w] for i in range(0, len(flat), w)]


class SplitMix64:
    """Sequence probe of the library's SplitMix64: returns, per draw,
    (next_u64, next_double, exponential(3.5), pareto(1.25, 0.2), uniform_int(-3, 17))."""

    @staticmethod
    def draws(seed: int, count: int = 4, tag: int | None = None):
        r = _call({"max_batch": 1, "components": [], "dnns": []}, "rng", (), seed=seed, count=count,
                  tag=tag)
        out = []
        for i in range(0, len(r), 5):
            out.append((int(r[i], 16), f64(r[i + 1]), f64(r[i + 2]), f64(r[i + 3]), r[i + 4]))
        return out


def generate_arrivals(process="poisson", rate=100.0, count=50, seed=1, dnn_mix=None):
    r = _call({"max_batch": 1, "components": [], "dnns": []}, "arrivals", (), process=process,
              rate=rate, count=count, seed=seed, dnn_mix=dnn_mix)
    return [(f64(t), d, bits) for t, d, bits in r]


def run_sim(job: dict) -> list[dict]:
    """Runs a {"job": "sim", ...} description; returns the JSONL records."""
    return [json.loads(l) for l in host_call(dict(job, job="sim")).splitlines()]
