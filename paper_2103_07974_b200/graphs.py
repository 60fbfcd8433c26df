"""Whole-rotation CUDA graphs: the crossover step replayed without the host.

For small apps the eager pipeline is host-bound: BASELINE config 1 (two MLP 784-256-10 jobs,
batch 64) has ~10 us of math per iteration but ~30 kernel launches plus autograd and the sync's
launches behind it, so the GPU idles between kernels and overlapping one app's sync with the other
app's compute gains nothing.  :class:`RotationGraph` captures one rotation of every registered app --
both streams, the events between them, K1 / C1 / K2 -- as ONE CUDA graph and replays it per rotation
(one launch per rotation), keeping the reference's semantics (scheduler.py:141-193):

crossover (Alg. 1), steady state, replay t::

    comm stream:    sync(N-1, t-1) | sync(0, t) | sync(1, t) | ... | sync(N-2, t)      (FIFO NIC lane)
    compute stream: compute(0, t) -> compute(1, t) -> ... -> [wait sync(N-1, t-1)] compute(N-1, t)

Every sync(j, t) waits for compute(j, t) (an event edge inside the graph); compute(j, t) for
j < N-1 needs sync(j, t-1), which ran in the previous replay (replays on one stream run back to
back), and compute(N-1, t) waits for the prologue sync(N-1, t-1) explicitly.  The last app's sync is
*deferred into the next replay* so that it overlaps the first app's compute of the next rotation --
the rotation boundary is no barrier.  Graph replays serialise, so compute(0, t+1) also waits for
sync(N-2, t); with rho <= 1 that sync ends inside compute(N-1, t) anyway (FIFO lane).
Sequential policy: compute(j, t) -> sync(j, t) -> compute(j+1, t) ..., all in one replay.

Graph layout differences from eager ``step()``: K1 (pack) runs on the compute stream right after
the backward -- so the deferred sync reads the app's own bucket (a fixed address) instead of the
graph's gradient buffers -- and the sync is C1 + K2 (``FusedGradientSync.sync_packed``).  Batches come
from ``App.data_graph(t_dev, worker)`` with the iteration in a device counter incremented by the
graph itself.  Every transport is capturable: bucket (NCCL all-reduce, or W simulated workers on one
GPU), sharded (NCCL RS/AG), and the peer transports p2p / ce, whose flag barriers are constant-valued
and self-resetting stream memory operations (cs_flag_barrier) and whose copy-engine pulls become
memcpy nodes; the adaptive transport is frozen at its calibrated choice.  Spans are not
recorded per phase inside replays (one graph launch per rotation); :meth:`phase_times` measures
each app's compute and sync as separate graphs instead.
"""

from __future__ import annotations

import contextlib
import statistics

import torch

from .errors import ConfigError
from .scheduler import CrossoverScheduler, Policy

__all__ = ["RotationGraph"]


class RotationGraph:
    """One CUDA graph per rotation for a registered :class:`CrossoverScheduler`.

    Usage: step the scheduler eagerly for at least two rotations (t = 1 bypasses Alg. 1's wait and
    initialises momentum; kernels and the allocator warm up), then ``begin()``, ``replay()`` once per
    rotation, ``end()`` -- after which ``sched.drain()`` / ``run``-style accounting applies."""

    def __init__(self, sched: CrossoverScheduler, rotations: int = 1):
        if not sched.states:
            raise ConfigError("no apps registered")
        for st in sched.states:
            if st.app.data_graph is None:
                raise ConfigError(f"job {st.job_id!r}: graph mode needs App.data_graph")
            if st.sync.mode not in ("bucket", "sharded", "p2p", "ce", "adaptive", "nvls"):
                raise ConfigError(f"job {st.job_id!r}: graph mode needs a bucket transport "
                                  f"(got {st.sync.mode!r})")
            if st.sync.snapshot is not None:
                raise ConfigError("graph mode does not record per-iteration weights")
        if sched.timer is not None:
            raise ConfigError("graph mode has no per-kernel timer (use phase_times)")
        its = {st.next_iteration for st in sched.states}
        if len(its) != 1 or min(its) < 3:
            raise ConfigError("graph mode starts after >= 2 eager rotations of every app")
        if rotations < 1:
            raise ConfigError("rotations per graph must be >= 1")
        self.sched = sched
        self.rotations = int(rotations)   # rotations unrolled into one graph (fewer launches)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=sched.device)
        self.graph: torch.cuda.CUDAGraph | None = None
        self.t = 0                # last iteration whose compute has been enqueued
        self.replays = 0
        self._keep = []           # tensors the graph reads / writes (static addresses)

    # -- pieces -------------------------------------------------------------------------------
    def _compute(self, st) -> None:
        """fwd / bwd of every local worker from data_graph(t_dev) + K1 into the app's bucket, on
        the current (compute) stream."""
        app = st.app
        sched = self.sched
        workers = [sched.rank * app.local_workers + w for w in range(app.local_workers)]
        amp = (torch.autocast("cuda", dtype=app.autocast_dtype, cache_enabled=False)
               if app.autocast_dtype else contextlib.nullcontext())
        with amp:
            losses = [app.loss_fn(app.model, app.data_graph(self.t_dev, w)) for w in workers]
        grads = [list(torch.autograd.grad(loss, app.params, allow_unused=True)) for loss in losses]
        st.sync.pack(grads, torch.cuda.current_stream().cuda_stream)
        st.graph_loss = losses[0]
        self._keep.append((losses, grads))

    def _sync(self, st) -> None:
        st.sync.sync_packed(self.sched.comm_stream.cuda_stream)

    # -- protocol -----------------------------------------------------------------------------
    def begin(self) -> None:
        """Enqueue rotation t0 (the first not yet stepped) eagerly in graph layout -- for
        crossover with the last app's sync deferred -- and capture the steady-state rotation."""
        sched = self.sched
        cs, ms = sched.compute_stream, sched.comm_stream
        states = sched.states
        n = len(states)
        t0 = states[0].next_iteration
        if t0 > min(st.app.iterations for st in states):
            raise ConfigError("no iterations left for graph mode")
        with torch.cuda.stream(cs):
            self.t_dev.fill_(t0)
            for j, st in enumerate(states):
                if sched.policy is Policy.CROSSOVER:
                    cs.wait_event(st.update_done)
                elif sched._last_update is not None:
                    cs.wait_event(sched._last_update)
                self._compute(st)
                if sched.policy is Policy.CROSSOVER and j == n - 1:
                    continue           # deferred into the first replay
                e = torch.cuda.Event()
                e.record(cs)
                ms.wait_event(e)
                with torch.cuda.stream(ms):
                    self._sync(st)
                done = torch.cuda.Event()
                done.record(ms)
                st.update_done = sched._last_update = done
        self.t = t0
        # the first replay's graph-internal comm branch must follow the eager syncs above
        tail = torch.cuda.Event()
        tail.record(ms)
        cs.wait_event(tail)
        self._capture()

    def _capture(self) -> None:
        sched = self.sched
        cs, ms = sched.compute_stream, sched.comm_stream
        states = sched.states
        n = len(states)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(self.rotations):
                self._capture_rotation(states, n)
        self.graph = g

    def _capture_rotation(self, states, n: int) -> None:
        """One rotation's nodes; it ends with the compute stream joining the comm stream, so a
        second copy in the same graph starts exactly where the next replay would."""
        sched = self.sched
        cs, ms = sched.compute_stream, sched.comm_stream
        self.t_dev.add_(1)
        fork = torch.cuda.Event()
        fork.record(cs)
        ms.wait_event(fork)
        if sched.policy is Policy.CROSSOVER:
            with torch.cuda.stream(ms):
                self._sync(states[n - 1])        # sync(N-1, t-1): the deferred one
            tail = torch.cuda.Event()
            tail.record(ms)
            for j, st in enumerate(states):
                if j == n - 1:
                    cs.wait_event(tail)          # Alg. 1: compute(N-1, t) after sync(N-1, t-1)
                self._compute(st)
                if j < n - 1:
                    e = torch.cuda.Event()
                    e.record(cs)
                    ms.wait_event(e)
                    with torch.cuda.stream(ms):
                        self._sync(st)
        else:
            for st in states:
                self._compute(st)
                e = torch.cuda.Event()
                e.record(cs)
                ms.wait_event(e)
                with torch.cuda.stream(ms):
                    self._sync(st)
                back = torch.cuda.Event()
                back.record(ms)
                cs.wait_event(back)
        join = torch.cuda.Event()
        join.record(ms)
        cs.wait_event(join)

    def replay(self) -> None:
        """`rotations` rotations: every app computes iterations t+1 .. t+rotations (and the syncs of
        the schedule above)."""
        if self.graph is None:
            raise ConfigError("begin() first")
        if self.t + self.rotations > min(st.app.iterations for st in self.sched.states):
            raise ConfigError("iteration budget exhausted")
        with torch.cuda.stream(self.sched.compute_stream):
            self.graph.replay()
        self.t += self.rotations
        self.replays += 1

    def end(self) -> None:
        """Drain: the last app's deferred sync (crossover), then hand the state back."""
        sched = self.sched
        cs, ms = sched.compute_stream, sched.comm_stream
        if sched.policy is Policy.CROSSOVER:
            e = torch.cuda.Event()
            e.record(cs)
            ms.wait_event(e)
            with torch.cuda.stream(ms):
                self._sync(sched.states[-1])
        done = torch.cuda.Event()
        done.record(ms)
        for st in sched.states:
            st.next_iteration = self.t + 1
            st.update_done = done
            st.awaiting_sync = True
            st.sync_of_iteration = self.t
            st.held = None
        sched._last_update = done

    def release(self) -> None:
        """Destroy the captured graph (and the references it keeps).  Required before the NCCL
        communicator it captured collectives of is destroyed: ncclCommDestroy waits for graphs
        that still hold NCCL work."""
        if self.graph is not None:
            torch.cuda.synchronize()
            self.graph.reset()
            self.graph = None
        self._keep.clear()

    # -- measurement ----------------------------------------------------------------------------
    def phase_times(self, reps: int = 20) -> tuple[list[float], list[float]]:
        """Device time (ms, median of `reps` back-to-back replays) of every app's compute graph
        (fwd / bwd + K1) and sync graph (C1 + K2), each captured alone -- the comp / comm of the
        overlap roofline in graph mode.  Parameters and momentum buffers are restored afterwards
        (the sync graphs apply extra updates while they are timed)."""
        sched = self.sched
        cs = sched.compute_stream
        torch.cuda.synchronize()
        saved = [[p.detach().clone() for p in st.app.params] for st in sched.states]
        saved_m = [[m.clone() for m in (st.sync.momentum_bufs or [])] for st in sched.states]
        comps, comms = [], []
        for st in sched.states:
            out = []
            for piece in ("compute", "sync"):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    if piece == "compute":
                        self._compute(st)
                    else:
                        st.sync.sync_packed(cs.cuda_stream)
                ts = []
                with torch.cuda.stream(cs):
                    for k in range(reps + 3):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(cs)
                        g.replay()
                        b.record(cs)
                        if k >= 3:
                            ts.append((a, b))
                torch.cuda.synchronize()
                out.append(statistics.median(a.elapsed_time(b) for a, b in ts))
                del g
            comps.append(out[0])
            comms.append(out[1])
        with torch.no_grad():
            for st, ps, ms_ in zip(sched.states, saved, saved_m):
                for p, s in zip(st.app.params, ps):
                    p.copy_(s)
                for m, s in zip(st.sync.momentum_bufs or [], ms_):
                    m.copy_(s)
        torch.cuda.synchronize()
        return comps, comms
