"""The crossover scheduler as a device pipeline of CUDA streams and events.

Reference: colosim.scheduler (scheduler.py:55-258) -- a rotation driver over one
GPU lane and one NIC lane, with two policies:

* ``crossover`` (Alg. 1, scheduler.py:141-174): apps take turns on the GPU in
  plan order; when app j's backward ends its fused gradient is queued on the
  NIC and the GPU moves on to app j+1, so j's sync overlaps j+1's compute.
  Compute (j, t) may start only after sync (j, t-1) completed (bypassed at
  t = 1); if the head app is not ready the GPU idles -- it never skips ahead.
* ``sequential`` (scheduler.py:177-193): compute, then sync to completion while
  the GPU idles, then the next app.

Device mapping (one process per GPU, every rank hosts every app):

  compute stream  (lane gpu0):  [wait update_done[j]]  fwd(j,t)  bwd(j,t)  record bwd_done
  comm stream     (lane nic0):  wait bwd_done  K1 pack -> C1 NCCL all-reduce -> K2 update
                                record update_done[j]

The single comm stream is the reference's single FIFO NIC lane shared by all
apps: a later app's sync can never overtake an earlier one, which
is what makes strict head-of-line stalling equivalent to the reference even
when one app's sync is long.  The host only enqueues; it never blocks inside
``step()``.  The emitted span order -- compute (j, t) then sync (j, t), slot by
slot in rotation order -- is the reference's append order (engine.py:146) and is
returned as a measured ``Trace``.
"""

from __future__ import annotations

import collections
import contextlib
import gc
import time
from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction
from typing import Any, Callable, Sequence

import torch

from .comm import NcclCommunicator
from .engine import GPU_LANE_ID, NIC_LANE_ID, Phase, SpanRecorder, Trace
from .errors import ConfigError, DeadlockError
from .fusion import FusedGradientSync, SgdSettings
from .workload import JobProfile

__all__ = [
    "Policy",
    "App",
    "SchedulePlan",
    "JobRuntimeState",
    "CrossoverScheduler",
    "simulate",
    "schedule_crossover",
    "schedule_sequential",
    "rotation_schedule",
    "steady_state_period",
    "predicted_speedup",
    "overlap_roofline",
    "GPU_LANE_ID",
    "NIC_LANE_ID",
]


class Policy(Enum):
    CROSSOVER = "crossover"
    SEQUENTIAL = "sequential"


@dataclass
class App:
    """A co-located data-parallel training app (the device analogue of JobProfile).

    ``loss_fn(model, batch)`` runs the forward pass and returns a scalar loss;
    ``data(iteration, worker)`` returns that worker's batch for iteration t
    (1-based; ``worker`` is the global worker index = rank * local_workers + w)
    as a tuple of tensors, either already on the device or in (pinned) host
    memory -- host batches are copied on a dedicated H2D stream.
    """

    job_id: str
    model: torch.nn.Module
    loss_fn: Callable[[torch.nn.Module, Any], torch.Tensor]
    data: Callable[[int, int], Sequence[torch.Tensor]]
    sgd: SgdSettings
    iterations: int
    local_workers: int = 1
    autocast_dtype: torch.dtype | None = None
    params: list[torch.Tensor] | None = None
    samples_per_batch: int = 0   # for samples/s accounting (per worker)
    autocast_cache: bool = True  # must be False when the model replays CUDA graphs
    flat_params: torch.Tensor | None = None   # set by fusion.flatten_parameters (sharded sync)
    # data_graph(t_dev, worker): the same batch as data(t, worker) with t read from a 1-element
    # int64 device tensor -- what lets a rotation be captured once and replayed (graphs.py)
    data_graph: Callable[[torch.Tensor, int], Sequence[torch.Tensor]] | None = None

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError(f"job {self.job_id!r}: iterations must be >= 1")
        if self.params is None:
            self.params = [p for p in self.model.parameters() if p.requires_grad]


@dataclass(frozen=True)
class SchedulePlan:
    """Ordered apps sharing the GPU(s) plus the policy (scheduler.py:60-77).

    Job order is the rotation order.  ``jobs`` may hold :class:`App` objects
    (device execution) or reference ``JobProfile`` records (schedule-only).
    """

    policy: Policy
    jobs: tuple
    cluster: Any = None

    def __post_init__(self):
        object.__setattr__(self, "jobs", tuple(self.jobs))
        if not self.jobs:
            raise ValueError("plan must contain at least one job")
        ids = [j.job_id for j in self.jobs]
        if len(set(ids)) != len(ids):
            raise ValueError("job ids must be unique within a plan")


@dataclass
class JobRuntimeState:
    """Per-app bookkeeping of the rotation driver (scheduler.py:80-87) + device state."""

    job_id: str
    next_iteration: int = 1
    awaiting_sync: bool = False
    sync_of_iteration: int = 0
    # device side
    app: App | None = None
    sync: FusedGradientSync | None = None
    update_done: Any = None          # torch.cuda.Event of the last K2
    held: Any = None                 # gradients still read by the comm stream
    losses: list = field(default_factory=list)


def rotation_schedule(job_order: Sequence[str], iterations: Sequence[int]) -> list[tuple[str, str, str, int]]:
    """The emitted phase schedule for a plan, as the device pipeline issues it.

    Rotation in plan order from a cursor, skipping exhausted apps
    (scheduler.py:106-115); each dispatched slot emits forward, backward on the
    GPU lane then the sync on the NIC lane (scheduler.py:117-128).  The order is
    a pure function of (job order, budgets) -- identical for both policies.
    """
    done = {j: 0 for j in job_order}
    budget = dict(zip(job_order, iterations))
    out = []
    n = len(job_order)
    cursor = 0
    remaining = sum(iterations)
    while remaining:
        for k in range(n):
            j = job_order[(cursor + k) % n]
            if done[j] < budget[j]:
                cursor = (cursor + k) % n
                break
        j = job_order[cursor]
        t = done[j] + 1
        out += [(GPU_LANE_ID, j, "forward", t), (GPU_LANE_ID, j, "backward", t),
                (NIC_LANE_ID, j, "sync", t)]
        done[j] = t
        remaining -= 1
        cursor = (cursor + 1) % n
    return out


class _KernelTimer:
    """CUDA-event brackets around K1/C1/K2 on the comm stream (for the roofline)."""

    def __init__(self, stream):
        self.stream = stream
        self.records: list[tuple[str, Any, Any]] = []
        self._open: dict[str, Any] = {}

    def begin(self, name: str) -> None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        self._open[name] = ev

    def end(self, name: str) -> None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        self.records.append((name, self._open.pop(name), ev))

    def summary(self) -> dict[str, list[float]]:
        out: dict[str, list[float]] = {}
        for name, a, b in self.records:
            b.synchronize()
            out.setdefault(name, []).append(a.elapsed_time(b))
        return out

    def clear(self) -> None:
        self.records.clear()


class CrossoverScheduler:
    """Registers co-located apps and steps them under crossover or sequential sync.

    One instance per process (= per GPU).  ``step()`` dispatches one rotation
    slot (one app's forward+backward plus its sync) and returns immediately;
    ``run()`` steps until every app exhausted its budget and returns the
    measured trace.
    """

    def __init__(self, policy: Policy = Policy.CROSSOVER, device: torch.device | int | None = None,
                 comm: NcclCommunicator | None = None, record_spans: bool = True,
                 record_weights: bool = False, align: int = 32, sync_mode: str = "auto",
                 time_kernels: bool = False, comm_priority: int = -1,
                 perturb: tuple[int, int] | None = None, watchdog_s: float | None = 600.0,
                 nvtx: bool = False, p2p_ctas: int | None = None, barrier: str = "auto",
                 sync_ctas: int | str | None = None, pack_engine: str = "sm"):
        if not torch.cuda.is_available():
            raise ConfigError("CrossoverScheduler needs a CUDA device (there is no CPU fallback)")
        if not isinstance(policy, Policy):
            raise ValueError("policy must be a Policy")
        self.policy = policy
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else (device.index if isinstance(device, torch.device) else device))
        self.comm = comm
        self.rank = comm.rank if comm is not None else 0
        self.align = align
        self.sync_mode = sync_mode
        self.record_weights = record_weights
        self.perturb = perturb
        self.watchdog_s = watchdog_s
        self.nvtx = nvtx
        self.p2p_ctas = p2p_ctas
        self.sync_ctas = sync_ctas
        self.pack_engine = pack_engine
        self.barrier = barrier
        with torch.cuda.device(self.device):
            self.compute_stream = torch.cuda.Stream(self.device)
            lo, hi = torch.cuda.Stream.priority_range()
            prio = max(hi, min(lo, comm_priority))
            self.comm_stream = torch.cuda.Stream(self.device, priority=prio)
            self.h2d_stream = torch.cuda.Stream(self.device)
            # the caching allocator keeps per-stream pools: give each stream a small- and a
            # large-block segment now, so the first iteration's allocations do not stall the host
            # in cudaMalloc while the device idles (it would stretch the first forward's span)
            for st_ in (self.compute_stream, self.comm_stream, self.h2d_stream):
                with torch.cuda.stream(st_):
                    torch.empty(256, dtype=torch.uint8, device=self.device)
                    torch.empty(4 << 20, dtype=torch.uint8, device=self.device)
        self.recorder = SpanRecorder(torch, record_spans)
        self.timer = _KernelTimer(self.comm_stream) if time_kernels else None
        self.states: list[JobRuntimeState] = []
        self.cursor = 0
        self._last_update = None
        self._started = False
        self._slot = 0
        self.tuner: _TransportTuner | None = None
        self.failed = False
        self.grid_choice: dict | None = None
        self._last_compute_start = None
        self._inflight: collections.deque = collections.deque()

    # -- registration (≙ building a SchedulePlan of JobProfiles) -------------
    def register(self, app: App) -> JobRuntimeState:
        if self._started:
            raise ConfigError("register every app before the first step()")
        if any(s.job_id == app.job_id for s in self.states):
            raise ValueError("job ids must be unique within a plan")
        for p in app.params:
            if p.device != self.device:
                raise ConfigError(f"job {app.job_id!r}: parameters must be on {self.device}")
        # SM footprint of the fused P2P / NVLS sync: under crossover it overlaps another app's
        # compute and has that compute as slack, so it holds few SMs (32 CTAs, ~NCCL's channel
        # count; 64 for nvls, whose multimem.ld_reduce round trips through the switch need more
        # loads in flight: 32 CTAs reach 0.58 of the W = 2 ceiling, 64 reach it,
        # tools/nvls_ceiling.cu); the sequential baseline runs it alone on the whole GPU.
        mode = self._mode_for(app)
        p2p_ctas = self.p2p_ctas if self.p2p_ctas is not None else (
            (64 if mode == "nvls" else 32) if self.policy is Policy.CROSSOVER else 0)
        sync = FusedGradientSync(app.params, app.sgd, self.comm, app.local_workers, self.align,
                                 mode, app.iterations if self.record_weights else 0,
                                 flat_params=app.flat_params, p2p_ctas=p2p_ctas,
                                 barrier=self.barrier, sync_ctas=self._sync_grid(),
                                 pack_engine=self.pack_engine)
        st = JobRuntimeState(app.job_id, app=app, sync=sync)
        self.states.append(st)
        return st

    def _sync_grid(self) -> int:
        """K1 / K2 grid cap.  Explicit value, else: one CTA per chunk (0).  A persistent cap
        (e.g. 2 x SM count) keeps a high-priority sync from holding back the other app's CTAs
        (see cs_pack in include/crossover.h); ``sync_ctas=-1`` asks for 2 CTAs per SM;
        ``sync_ctas="auto"`` starts at 0 and lets :meth:`calibrate_grid` measure the choice."""
        if self.sync_ctas is None or self.sync_ctas == "auto":
            return 0
        if self.sync_ctas < 0:
            return 2 * torch.cuda.get_device_properties(self.device).multi_processor_count
        return int(self.sync_ctas)

    def _mode_for(self, app: App) -> str:
        """Transport per policy when the caller left it to us.

        With peer-mappable flat parameters at W > 1: under crossover the sync overlaps another
        app's compute, so it goes through the copy engines ("ce": NVLink pulls that hold no SM,
        ~1-6 % GEMM slowdown vs 15-100 % for SM-driven collectives, tools/cebench.py) unless it
        no longer fits under the other apps' compute -- the copy engines move fewer bytes per
        second than the P2P kernel -- so the crossover run is "adaptive" (:class:`_TransportTuner`
        measures both and keeps the faster); the sequential baseline has the GPU to itself and
        takes the fastest isolated path, the fused P2P kernel on the full grid.  Every transport
        sums in rank order, so the weights are bitwise identical whichever runs.  Flat parameters
        bound to an NVSwitch multicast object (flatten_parameters(ipc="nvls")) select the nvls
        transport for both policies."""
        if self.sync_mode != "auto" or self.comm is None or self.comm.world < 2:
            return self.sync_mode
        from .nvls import nvls_buffer_of
        from .p2p import buffer_of

        if app.flat_params is not None and app.local_workers == 1 and nvls_buffer_of(app.flat_params) is not None:
            return "nvls"          # multicast-bound flat parameters: the switch reduces and broadcasts
        if app.flat_params is None or buffer_of(app.flat_params) is None or app.local_workers != 1:
            return self.sync_mode
        return "adaptive" if self.policy is Policy.CROSSOVER else "p2p"

    @property
    def job_order(self) -> list[str]:
        return [s.job_id for s in self.states]

    # -- rotation (scheduler.py:106-122) -------------------------------------
    def _next_with_work(self) -> JobRuntimeState | None:
        n = len(self.states)
        for k in range(n):
            probe = (self.cursor + k) % n
            st = self.states[probe]
            if st.next_iteration <= st.app.iterations:
                self.cursor = probe
                return st
        return None

    def pending(self) -> list[tuple[str, int]]:
        out = []
        for st in self.states:
            if st.next_iteration <= st.app.iterations:
                out.append((st.job_id, st.next_iteration))
        return out

    def _to_device(self, batch: Sequence[torch.Tensor]) -> tuple:
        if all(not isinstance(x, torch.Tensor) or x.device == self.device for x in batch):
            return tuple(batch)
        with torch.cuda.stream(self.h2d_stream):
            dev = tuple(x.to(self.device, non_blocking=True) if isinstance(x, torch.Tensor) else x
                        for x in batch)
        ev = torch.cuda.Event()
        ev.record(self.h2d_stream)
        self.compute_stream.wait_event(ev)
        for x in dev:
            if isinstance(x, torch.Tensor):
                x.record_stream(self.compute_stream)
        return dev

    def step(self) -> bool:
        """Dispatch one rotation slot; False once every app is exhausted."""
        if not self.states:
            raise ConfigError("no apps registered")
        if not self._started:
            self._start()
        st = self._next_with_work()
        if st is None:
            return False
        app, t = st.app, st.next_iteration
        cs, ms = self.compute_stream, self.comm_stream
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        self._slot += 1
        if self.tuner is not None:
            st.sync.set_transport(self.tuner.transport)

        with torch.cuda.stream(cs):
            # Alg. 1 readiness (scheduler.py:158): compute (j, t) after sync (j, t-1).
            if self.policy is Policy.CROSSOVER:
                if t > 1:
                    cs.wait_event(st.update_done)
            elif self._last_update is not None:
                # sequential baseline: the GPU idles until the previous sync completed
                cs.wait_event(self._last_update)
            # stream-ordered after this app's own K2, so the caching allocator may
            # now reuse the previous iteration's gradient memory on this stream
            st.held = None
            workers = [self.rank * app.local_workers + w for w in range(app.local_workers)]
            batches = [self._to_device(app.data(t, w)) for w in workers]
            e_f0 = ev()
            e_f0.record(cs)
            self._last_compute_start = e_f0
            amp = (torch.autocast("cuda", dtype=app.autocast_dtype, cache_enabled=app.autocast_cache)
                   if app.autocast_dtype else contextlib.nullcontext())
            losses = []
            with amp, self._range(f"{st.job_id} forward t{t}"):
                for b in batches:
                    losses.append(app.loss_fn(app.model, b))
            e_f1 = ev()
            e_f1.record(cs)
            with self._range(f"{st.job_id} backward t{t}"):
                grads = [list(torch.autograd.grad(loss, app.params, allow_unused=True))
                         for loss in losses]
            e_b1 = ev()
            e_b1.record(cs)
        st.losses.append(losses[0].detach())
        st.held = grads
        st.awaiting_sync, st.sync_of_iteration = True, t

        with torch.cuda.stream(ms):
            ms.wait_event(e_b1)
            e_s0 = ev()
            e_s0.record(ms)
            with self._range(f"{st.job_id} sync t{t}"):
                st.sync.sync(grads, ms.cuda_stream, t - 1 if self.record_weights else None, self.timer)
            if self.perturb is not None and self.perturb == (self.job_index(st.job_id), t):
                _nudge_first_coordinate(app.params[0], st.sync, t - 1 if self.record_weights else None)
            e_s1 = ev()
            e_s1.record(ms)
        st.update_done = e_s1
        self._last_update = e_s1
        # syncs still in flight, oldest first (failure reports name the oldest unfinished one);
        # only the head is queried, so this stays O(1) per step
        self._inflight.append((st.job_id, t, e_s1))
        while len(self._inflight) > 1 and self._inflight[0][2].query():
            self._inflight.popleft()

        self.recorder.add(GPU_LANE_ID, st.job_id, Phase.FORWARD, t, e_f0, e_f1)
        self.recorder.add(GPU_LANE_ID, st.job_id, Phase.BACKWARD, t, e_f1, e_b1)
        self.recorder.add(NIC_LANE_ID, st.job_id, Phase.SYNC, t, e_s0, e_s1)
        st.next_iteration = t + 1
        self.cursor = (self.cursor + 1) % len(self.states)
        return True

    def _start(self) -> None:
        self._started = True
        self.recorder.start(self.compute_stream)
        adaptive = [s.sync.mode == "adaptive" for s in self.states]
        if all(adaptive):
            self.tuner = _TransportTuner()
        elif any(adaptive):
            raise ConfigError("adaptive transport must be used by every app or none")

    def calibrate(self, rotations: int = 4) -> dict | None:
        """Measured choice of the adaptive transport (copy engines vs the fused P2P kernel).

        Steps ``rotations`` rotations over the copy engines and ``rotations + 1`` with the P2P
        kernel -- real training iterations: both transports sum the W shards in rank order with the
        same update rule, so the weights are bitwise those of either transport -- then waits for the
        device (here, outside ``step()``, which never blocks), takes each transport's median
        rotation period between compute starts (the first rotation of each window is a warm-up),
        sums the medians over the ranks and keeps the faster transport on every rank.  Returns the
        tuner summary, or None when the plan is not adaptive or too short (stays on the copy
        engines).  ``run()`` calls it first when every budget allows."""
        if not self._started:
            self._start()
        if self.tuner is None or self.tuner.decided:
            return None if self.tuner is None else self.tuner.summary()
        need = 2 * rotations + 1
        if rotations < 2 or any(st.app.iterations - st.next_iteration + 1 < need for st in self.states):
            return None
        starts = {}
        for k in range(need):
            self.tuner.transport = "ce" if k < rotations else "p2p"
            for j in range(len(self.states)):
                self.step()
                if j == 0:
                    starts[k] = self._last_compute_start
        # one more rotation boundary: the first compute after the last p2p rotation is enqueued by
        # the caller's next step(); the window's last start is that of rotation 2R (already issued)
        starts[need - 1].synchronize()
        ce = sorted(starts[k].elapsed_time(starts[k + 1]) for k in range(1, rotations))
        p2p = sorted(starts[k].elapsed_time(starts[k + 1]) for k in range(rotations + 1, need - 1))
        medians = [ce[len(ce) // 2], p2p[len(p2p) // 2]]
        self.tuner.decide(medians, self.comm)
        return self.tuner.summary()

    def calibrate_grid(self, rotations: int = 3, candidates: Sequence[int] | None = None) -> dict | None:
        """Measured K1 / K2 grid cap for ``sync_ctas="auto"``.

        A sync kernel on the high-priority comm stream with one CTA per chunk grabs every SM as
        the other app's CTAs retire, so a tensor-core GEMM pays almost its whole duration; a
        persistent grid of a few dozen CTAs co-resides with the GEMM's CTAs (a B200 SM holding
        one 256-thread, 168-register GEMM CTA still has room for one K2 CTA) and costs the GEMM
        ~10 % of K2's time, but runs 3-6x longer -- the right choice only while the sync has
        slack under the other apps' compute (tools/k2_interference.py).  So it is measured like
        the transport: every candidate cap (default: one CTA per chunk, one CTA per SM, 64, 32)
        runs ``rotations + 1`` real rotations (the grid never changes the results), the median
        period of each window's last ``rotations`` rotations is summed over the ranks, and every
        rank keeps the fastest cap.  Host waits only here, outside ``step()``."""
        if not self._started:
            self._start()
        if self.sync_ctas != "auto" or self.grid_choice is not None:
            return self.grid_choice
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        cands = list(candidates) if candidates is not None else [0, sms, 64, 32]
        per = rotations + 1
        need = len(cands) * per + 1
        if rotations < 2 or any(st.app.iterations - st.next_iteration + 1 < need for st in self.states):
            return None
        starts = []
        for k in range(need):
            cap = cands[min(k // per, len(cands) - 1)]
            for st in self.states:
                st.sync.sync_ctas = cap
            for j in range(len(self.states)):
                self.step()
                if j == 0:
                    starts.append(self._last_compute_start)
        starts[-1].synchronize()
        medians = []
        for i in range(len(cands)):
            r0 = i * per
            p = sorted(starts[k].elapsed_time(starts[k + 1]) for k in range(r0 + 1, r0 + per))
            medians.append(p[len(p) // 2])
        import torch.distributed as dist

        t = torch.tensor(medians, dtype=torch.float64)
        world = self.comm.world if self.comm is not None else 1
        if world > 1 and dist.is_initialized():
            if dist.get_backend() == "nccl":
                d = t.to(self.device)
                dist.all_reduce(d)
                t = d.cpu()
            else:
                dist.all_reduce(t)
        periods = [float(x) / world for x in t]
        best = min(range(len(cands)), key=lambda i: periods[i])
        for st in self.states:
            st.sync.sync_ctas = cands[best]
        self.grid_choice = {"choice": cands[best], "candidates": cands,
                            "period_ms": [round(x, 4) for x in periods]}
        return self.grid_choice

    def _range(self, name: str):
        """NVTX range around a phase (visible in Nsight Systems) when nvtx=True."""
        return torch.cuda.nvtx.range(name) if self.nvtx else contextlib.nullcontext()

    def job_index(self, job_id: str) -> int:
        return self.job_order.index(job_id)

    def drain(self, timeout_s: float | None = None) -> None:
        """Wait for the final syncs (the drain of Alg. 1) and release gradients.

        Failure detection: while waiting, NCCL's asynchronous error state is polled;
        an error, or no completion within ``timeout_s`` (default: ``self.watchdog_s``), aborts the
        communicator and raises DeadlockError(job, iteration) for the oldest unfinished sync --
        the device analogue of the reference's quiescence check (engine.py:168-173).
        """
        join = torch.cuda.Event()
        join.record(self.comm_stream)
        self.compute_stream.wait_event(join)
        done = torch.cuda.Event()
        done.record(self.compute_stream)
        limit = self.watchdog_s if timeout_s is None else timeout_s
        t0 = time.monotonic()
        while not done.query():
            if self.comm is not None:
                try:
                    self.comm.check_async_error()
                except RuntimeError as exc:
                    self._fail(f"NCCL error: {exc}")
            if limit is not None and time.monotonic() - t0 > limit:
                self._fail(f"no progress within {limit:.0f} s")
            time.sleep(0.0005)
        for st in self.states:
            st.held = None
            st.awaiting_sync = False
        if self.comm is not None:
            self.comm.check_async_error()

    def _fail(self, detail: str) -> None:
        """Failure path: unblock the device, then raise DeadlockError(job, iteration).

        NCCL kernels waiting for a dead peer end with ncclCommAbort; flag-barrier waits (stream
        memory operations, which no abort can cancel) are satisfied by writing 1 into the shared
        flag segments from the host, repeatedly until the comm stream drained.  The queued work then drains (its results are
        garbage and the syncs are marked failed), so later synchronize / teardown calls return."""
        pending = [(j, t) for j, t, e in self._inflight if not e.query()]
        job, it = pending[0] if pending else (self.states[0].job_id, self.states[0].next_iteration)
        if self.comm is not None:
            self.comm.abort()
        done = torch.cuda.Event()
        done.record(self.comm_stream)
        t0 = time.monotonic()
        while True:
            for st in self.states:          # a released wait resets its row: keep releasing
                st.sync.release_waits()
            if done.query() or time.monotonic() - t0 > 30.0:
                break
            time.sleep(0.001)
        self.failed = True
        raise DeadlockError(job, it, f"policy={self.policy.value}; {detail}")

    def run(self) -> Trace:
        """Step every app through its budget; returns the measured trace.

        Python's cyclic GC is paused while stepping: a collection pauses the host for tens of
        ms, the GPU queue drains meanwhile, and at W > 1 every rank then waits for the paused
        one at the next barrier."""
        was_enabled = gc.isenabled()
        gc.collect()
        gc.disable()
        try:
            if not self._started:
                self._start()
            if self.tuner is not None and self._slot == 0:
                self.calibrate()
            if self.sync_ctas == "auto" and self.grid_choice is None:
                self.calibrate_grid()
            while self.step():
                pass
        finally:
            if was_enabled:
                gc.enable()
        self.drain()
        stuck = self.pending()
        if stuck:
            raise DeadlockError(stuck[0][0], stuck[0][1], f"policy={self.policy.value}")
        return self.recorder.resolve()

    def weights(self, job_id: str) -> torch.Tensor:
        """[iterations, bucket] per-iteration weights captured by K2 (record_weights=True)."""
        st = self.states[self.job_index(job_id)]
        if st.sync.snapshot is None:
            raise ConfigError("record_weights=False")
        return st.sync.snapshot

    def close(self) -> None:
        """Release peer mappings (p2p sync); call after the last drain()."""
        for st in self.states:
            st.sync.close()

    @property
    def kernel_launches(self) -> int:
        return sum(s.sync.kernel_launches for s in self.states)


class _TransportTuner:
    """State of the adaptive transport (measured by :meth:`CrossoverScheduler.calibrate`).

    Until calibrated every sync runs over the copy engines; ``decide`` sums the per-rank median
    rotation periods of both transports over the ranks (host-side, after the device reached the
    end of the calibration window) so every rank keeps the same transport."""

    def __init__(self):
        self.transport = "ce"
        self.decided = False
        self.periods_ms: dict[str, float] | None = None

    def decide(self, medians: list[float], comm) -> None:
        import torch.distributed as dist

        world = comm.world if comm is not None else 1
        t = torch.tensor(medians, dtype=torch.float64)
        if world > 1 and dist.is_initialized():
            if dist.get_backend() == "nccl":
                d = t.to(torch.cuda.current_device())
                dist.all_reduce(d)
                t = d.cpu()
            else:
                dist.all_reduce(t)
        ce, p2p = (float(x) / world for x in t)
        self.periods_ms = {"ce": ce, "p2p": p2p}
        self.transport = "ce" if ce <= p2p else "p2p"
        self.decided = True

    @property
    def choice(self) -> str:
        return self.transport

    @property
    def active(self) -> bool:
        return self.decided

    def summary(self) -> dict:
        return {"active": self.decided, "choice": self.transport,
                "calibration_period_ms": self.periods_ms}


def _nudge_first_coordinate(param: torch.Tensor, sync: FusedGradientSync, row: int | None) -> None:
    """Fault-injection hook of run_crossover (equivalence.py:214-219): +1 ulp on p[0]."""
    with torch.no_grad():
        flat = torch.as_strided(param, (1,), (1,))
        flat.copy_(torch.nextafter(flat, torch.full_like(flat, float("inf"))))
        if row is not None:
            sync.snapshot[row, :1].copy_(flat)


# -- reference-shaped entry points --------------------------------------------

def _run_plan(plan: SchedulePlan, **kw) -> Trace:
    if not all(isinstance(j, App) for j in plan.jobs):
        raise ConfigError("device execution needs App jobs (JobProfile plans have no model)")
    sched = CrossoverScheduler(plan.policy, **kw)
    for app in plan.jobs:
        sched.register(app)
    try:
        return sched.run()
    except DeadlockError as exc:
        raise DeadlockError(exc.job_id, exc.iteration, f"policy={plan.policy.value}") from exc


def schedule_crossover(plan: SchedulePlan, **kw) -> Trace:
    """Run the plan on the device under Alg. 1 (scheduler.py:209-212)."""
    if plan.policy is not Policy.CROSSOVER:
        raise ValueError("plan.policy must be crossover")
    return _run_plan(plan, **kw)


def schedule_sequential(plan: SchedulePlan, **kw) -> Trace:
    """Run the plan on the device under the non-overlapped baseline (scheduler.py:215-218)."""
    if plan.policy is not Policy.SEQUENTIAL:
        raise ValueError("plan.policy must be sequential")
    return _run_plan(plan, **kw)


def simulate(plan: SchedulePlan, **kw) -> Trace:
    """Run the plan under its configured policy (scheduler.py:221-225)."""
    return schedule_crossover(plan, **kw) if plan.policy is Policy.CROSSOVER else schedule_sequential(plan, **kw)


# -- closed forms (scheduler.py:228-258) and the overlap roofline --------------

def _homogeneous(comps: Sequence[int], comms: Sequence[int]) -> tuple[int, int]:
    if len(set(comps)) != 1 or len(set(comms)) != 1:
        raise ValueError("closed forms require homogeneous jobs (equal compute and sync "
                         "durations); simulate heterogeneous plans instead")
    return comps[0], comms[0]


def steady_state_period(policy: Policy, comps: Sequence[int], comms: Sequence[int]) -> int:
    """N*max(comp, comm) under crossover, N*(comp+comm) sequential (homogeneous)."""
    comp, comm = _homogeneous(comps, comms)
    n = len(comps)
    return n * max(comp, comm) if policy is Policy.CROSSOVER else n * (comp + comm)


def predicted_speedup(comps: Sequence[int], comms: Sequence[int]) -> Fraction:
    """(comp + comm) / max(comp, comm) = 1 + rho while rho <= 1 (homogeneous)."""
    comp, comm = _homogeneous(comps, comms)
    return Fraction(comp + comm, max(comp, comm))


def overlap_roofline(comps: Sequence[float], comms: Sequence[float]) -> dict[str, float]:
    """Per-rotation lower bounds on the crossover period.

    ``north_star``: max(Σcomp, Σcomm).  ``tight``: the reference's bound that
    also includes maxᵢ(compᵢ + commᵢ) (tests/test_scheduler.py:260-269).
    ``sequential``: Σ(compᵢ + commᵢ), the back-to-back period.
    """
    s_comp, s_comm = float(sum(comps)), float(sum(comms))
    tight = max(s_comp, s_comm, max(c + m for c, m in zip(comps, comms)))
    return {"north_star": max(s_comp, s_comm), "tight": tight, "sequential": s_comp + s_comm}


def profile_of(app: App, forward_ns: int, backward_ns: int) -> JobProfile:
    """Reference JobProfile of a registered app with measured durations."""
    from .workload import tensor_specs_from_module

    fwd, bwd = max(int(forward_ns), 0), max(int(backward_ns), 0)
    if fwd + bwd == 0:
        bwd = 1  # JobProfile requires forward + backward > 0 (workload.py:61-62)
    return JobProfile(app.job_id, fwd, bwd, tensor_specs_from_module(app.model), app.iterations)
