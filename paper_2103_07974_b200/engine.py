"""Lanes, spans and traces of the device pipeline.

Reference: colosim.engine (engine.py:41-289).  The reference's lanes are
simulated resources with a ``busy_until`` clock; here they are CUDA streams:

  lane ``gpu0`` (LaneKind.COMPUTE) = the compute stream (forward/backward of every app)
  lane ``nic0`` (LaneKind.NETWORK) = the single comm stream (K1 pack -> C1 NCCL -> K2 update)

A stream is an exclusive FIFO lane exactly like ``Lane`` with ``busy_until``
(engine.py:141): work starts when the previous item finished and its wait
events fired.  Span times come from CUDA events recorded on the lane's stream
(``SpanRecorder``) and are converted to integer nanoseconds against one origin
event, so the same ``Span``/``Trace`` schema, the same legality checker and the
same JSON / Chrome-trace exports apply to measured GPU runs.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from enum import Enum

__all__ = [
    "LaneKind",
    "Phase",
    "EventKind",
    "Span",
    "Trace",
    "validate_trace",
    "trace_to_json",
    "trace_to_chrome_json",
    "schedule_key",
    "SpanRecorder",
    "GPU_LANE_ID",
    "NIC_LANE_ID",
]

GPU_LANE_ID = "gpu0"
NIC_LANE_ID = "nic0"


class LaneKind(Enum):
    COMPUTE = "compute"
    NETWORK = "network"


class Phase(Enum):
    FORWARD = "forward"
    BACKWARD = "backward"
    SYNC = "sync"


class EventKind(Enum):
    # value = same-time tie-break order (engine.py:52-56)
    COMPUTE_DONE = 0
    COMM_DONE = 1


@dataclass(frozen=True)
class Span:
    lane_id: str
    job_id: str
    phase: Phase
    iteration: int
    start: int
    end: int


@dataclass(frozen=True)
class Trace:
    spans: tuple[Span, ...]
    makespan: int


def schedule_key(trace: Trace) -> list[tuple[str, str, str, int]]:
    """The phase schedule: (lane, job, phase, iteration) in emission order.

    This is the object the north star requires to be bit-exact against the
    reference's ``schedule_crossover`` / ``schedule_sequential`` span order.
    """
    return [(s.lane_id, s.job_id, s.phase.value, s.iteration) for s in trace.spans]


def validate_trace(trace: Trace) -> list[str]:
    """Legality of a trace; empty list = legal.  Same rules as engine.py:178-242.

    1. every span has 0 <= start <= end;
    2. spans on one lane never overlap;
    3. per job: at most one span per (iteration, phase); forward and backward
       present for every iteration; sync present for every non-final iteration;
    4. per job and iteration: forward.end <= backward.start <= ...,
       sync.start >= backward.end, next forward.start >= this sync.end;
    5. makespan == max span end.
    """
    out: list[str] = []
    lanes: dict[str, list[Span]] = {}
    jobs: dict[str, dict[int, dict[Phase, Span]]] = {}
    for s in trace.spans:
        if s.start < 0 or s.end < s.start:
            out.append(f"span {s.lane_id}/{s.job_id}/{s.phase.value}/t{s.iteration}: "
                       f"bad interval [{s.start}, {s.end}]")
        lanes.setdefault(s.lane_id, []).append(s)
        slot = jobs.setdefault(s.job_id, {}).setdefault(s.iteration, {})
        if s.phase in slot:
            out.append(f"job {s.job_id}: duplicate {s.phase.value} span for iteration {s.iteration}")
        else:
            slot[s.phase] = s

    for lane_id, spans in lanes.items():
        spans = sorted(spans, key=lambda x: (x.start, x.end))
        for a, b in zip(spans, spans[1:]):
            if b.start < a.end:
                out.append(f"lane {lane_id}: {a.job_id}/t{a.iteration} [{a.start},{a.end}] "
                           f"overlaps {b.job_id}/t{b.iteration} [{b.start},{b.end}]")

    for job_id, iters in jobs.items():
        final = max(iters)
        prev_sync = None
        for t in sorted(iters):
            ph = iters[t]
            fwd, bwd, syn = ph.get(Phase.FORWARD), ph.get(Phase.BACKWARD), ph.get(Phase.SYNC)
            if fwd is None:
                out.append(f"job {job_id}: missing forward span for iteration {t}")
            if bwd is None:
                out.append(f"job {job_id}: missing backward span for iteration {t}")
            if syn is None and t < final:
                out.append(f"job {job_id}: missing sync span for iteration {t}")
            if fwd is not None and bwd is not None and bwd.start < fwd.end:
                out.append(f"job {job_id}: backward precedes forward at iteration {t}")
            if bwd is not None and syn is not None and syn.start < bwd.end:
                out.append(f"job {job_id}: sync starts before backward ends at iteration {t}")
            if prev_sync is not None and fwd is not None and fwd.start < prev_sync.end:
                out.append(f"job {job_id}: iteration {t} compute starts before "
                           f"iteration {prev_sync.iteration} sync completes")
            prev_sync = syn

    last = max((s.end for s in trace.spans), default=0)
    if trace.makespan != last:
        out.append(f"makespan {trace.makespan} != max span end {last}")
    return out


def trace_to_json(trace: Trace) -> str:
    """JSON array of span records (same keys as engine.py:245-258)."""
    rows = [{"lane_id": s.lane_id, "job_id": s.job_id, "phase": s.phase.value,
             "iteration": s.iteration, "start_ns": s.start, "end_ns": s.end}
            for s in trace.spans]
    return json.dumps(rows, indent=2) + "\n"


def trace_to_chrome_json(trace: Trace) -> str:
    """Chrome trace-event JSON: one row per lane, "X" events in microseconds."""
    lane_ids = sorted({s.lane_id for s in trace.spans})
    tid = {lane: i for i, lane in enumerate(lane_ids)}
    events = [{"name": "thread_name", "ph": "M", "pid": 0, "tid": tid[lane],
               "args": {"name": lane}} for lane in lane_ids]
    events += [{"name": f"{s.job_id} {s.phase.value} t{s.iteration}", "ph": "X",
                "ts": s.start / 1000.0, "dur": (s.end - s.start) / 1000.0, "pid": 0,
                "tid": tid[s.lane_id], "args": {"job": s.job_id, "iteration": s.iteration}}
               for s in trace.spans]
    return json.dumps({"traceEvents": events, "displayTimeUnit": "ms"}, indent=2) + "\n"


class SpanRecorder:
    """Records spans as pairs of CUDA events and resolves them into a Trace.

    ``origin`` is recorded on the compute stream before the first span; every
    span boundary is an event recorded on its lane's stream *after* the lane's
    cross-stream waits, so causality holds in the measured times by
    construction (sync.start >= backward.end; next forward.start >= sync.end).
    Resolving calls ``torch.cuda.Event.synchronize`` on the last event only.
    """

    def __init__(self, torch_mod, enabled: bool = True):
        self._torch = torch_mod
        self.enabled = enabled
        self._pending: list[tuple[str, str, Phase, int, object, object]] = []
        self.origin = None

    def event(self):
        return self._torch.cuda.Event(enable_timing=True)

    def start(self, stream) -> None:
        self._pending.clear()
        self.origin = self.event()
        self.origin.record(stream)

    def add(self, lane_id: str, job_id: str, phase: Phase, iteration: int, ev_start, ev_end) -> None:
        if self.enabled:
            self._pending.append((lane_id, job_id, phase, iteration, ev_start, ev_end))

    def resolve(self) -> Trace:
        if self.origin is None:
            return Trace((), 0)
        for item in self._pending:
            item[5].synchronize()
        spans = []
        for lane_id, job_id, phase, it, a, b in self._pending:
            t0 = round(self.origin.elapsed_time(a) * 1e6)
            t1 = round(self.origin.elapsed_time(b) * 1e6)
            spans.append(Span(lane_id, job_id, phase, it, int(t0), int(max(t0, t1))))
        makespan = max((s.end for s in spans), default=0)
        return Trace(tuple(spans), makespan)
