"""Queue-free restatement of the reference's crossover / sequential schedules.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reference semantics restated (paths under /root/reference/pkg/src/colosim):
  * rotation in plan order from a cursor, skipping exhausted jobs -- scheduler.py:106-115
  * one compute task = forward then backward, back to back on the GPU lane -- scheduler.py:117-122
  * at COMPUTE_DONE the sync is queued on the single FIFO NIC lane -- scheduler.py:124-128,
    engine.py:141 (start = max(busy_until, now))
  * crossover: compute (j, t) ready iff t == 1 or sync (j, t-1) done; otherwise the GPU
    idles on that job, never skipping ahead -- scheduler.py:151-174
  * sequential: next compute only after the current sync completed -- scheduler.py:177-193
  * spans are appended in enqueue order -- engine.py:146-147

Spans are (lane_id, job_id, phase, iteration, start, end) tuples; jobs are
(job_id, forward_ns, backward_ns, sync_ns, iterations) tuples.
"""

from __future__ import annotations

from fractions import Fraction

GPU = "gpu0"
NIC = "nic0"


def _next_job(jobs, done, cursor):
    n = len(jobs)
    for k in range(n):
        i = (cursor + k) % n
        if done[i] < jobs[i][4]:
            return i
    return None


def _dur(durations, job_id, phase, t, default):
    return default if durations is None else durations.get((job_id, phase, t), default)


def crossover(jobs, durations=None):
    """Spans (in emission order) and makespan of the Alg. 1 schedule.

    ``durations`` optionally overrides single phases: {(job_id, phase, t): ns} (e.g. measured
    span lengths, to predict the start times a device run must have had)."""
    gpu_free = nic_free = 0
    sync_end = [0] * len(jobs)
    done = [0] * len(jobs)
    spans = []
    cursor = 0
    while True:
        i = _next_job(jobs, done, cursor)
        if i is None:
            break
        job_id, fwd, bwd, comm, _ = jobs[i]
        t = done[i] + 1
        fwd, bwd = _dur(durations, job_id, "forward", t, fwd), _dur(durations, job_id, "backward", t, bwd)
        comm = _dur(durations, job_id, "sync", t, comm)
        start = max(gpu_free, sync_end[i] if t > 1 else 0)
        mid, end = start + fwd, start + fwd + bwd
        spans += [(GPU, job_id, "forward", t, start, mid), (GPU, job_id, "backward", t, mid, end)]
        gpu_free = end
        s0 = max(nic_free, end)
        nic_free = sync_end[i] = s0 + comm
        spans.append((NIC, job_id, "sync", t, s0, nic_free))
        done[i] = t
        cursor = (i + 1) % len(jobs)
    return spans, max((s[5] for s in spans), default=0)


def sequential(jobs, durations=None):
    """Spans and makespan of the non-overlapped baseline (``durations`` as in crossover)."""
    now = 0
    done = [0] * len(jobs)
    spans = []
    cursor = 0
    while True:
        i = _next_job(jobs, done, cursor)
        if i is None:
            break
        job_id, fwd, bwd, comm, _ = jobs[i]
        t = done[i] + 1
        fwd, bwd = _dur(durations, job_id, "forward", t, fwd), _dur(durations, job_id, "backward", t, bwd)
        comm = _dur(durations, job_id, "sync", t, comm)
        spans += [(GPU, job_id, "forward", t, now, now + fwd),
                  (GPU, job_id, "backward", t, now + fwd, now + fwd + bwd),
                  (NIC, job_id, "sync", t, now + fwd + bwd, now + fwd + bwd + comm)]
        now += fwd + bwd + comm
        done[i] = t
        cursor = (i + 1) % len(jobs)
    return spans, max((s[5] for s in spans), default=0)


def schedule_order(spans):
    """(lane, job, phase, iteration) in emission order -- the bit-exact schedule."""
    return [s[:4] for s in spans]


def crossover_period(jobs, max_rotations: int = 10_000) -> Fraction:
    """Exact asymptotic time per rotation (budgets ignored): detect the periodic regime."""
    gpu_free = nic_free = 0
    sync_end = [0] * len(jobs)
    seen: dict[tuple, tuple[int, int]] = {}
    for r in range(1, max_rotations + 1):
        for i, (_, fwd, bwd, comm, _) in enumerate(jobs):
            start = max(gpu_free, sync_end[i] if r > 1 else 0)
            gpu_free = start + fwd + bwd
            nic_free = sync_end[i] = max(nic_free, gpu_free) + comm
        key = (nic_free - gpu_free, *(e - gpu_free for e in sync_end))
        if key in seen:
            r0, g0 = seen[key]
            return Fraction(gpu_free - g0, r - r0)
        seen[key] = (r, gpu_free)
    raise AssertionError("no periodic regime")
