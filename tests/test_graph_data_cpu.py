"""Graph-mode batch selection on CPU: App.data_graph(t_dev, worker) must return exactly the batch
App.data(t, worker) returns (graphs.RotationGraph reads the iteration from a device counter), and
the queue-free schedule oracle must honour per-span duration overrides (the timing tests feed it
measured durations)."""

import numpy as np
import torch

from oracle import schedule as osched


def test_gather_data_graph_matches_eager():
    from paper_2103_07974_b200.apps import _GatherData

    g = torch.Generator().manual_seed(0)
    x = torch.randn(50, 7, generator=g)
    y = torch.randint(0, 10, (50,), generator=g)
    idx = torch.randint(0, 50, (6, 3, 4), generator=g)          # [T, workers, batch]
    d = _GatherData(x, y, idx)
    for t in range(1, 7):
        for w in range(3):
            a = d(t, w)
            b = d.graph(torch.tensor([t]), w)
            assert all(torch.equal(p, q) for p, q in zip(a, b))


def test_cycle_data_graph_keeps_channels_last():
    from paper_2103_07974_b200.apps import _CycleData

    g = torch.Generator().manual_seed(1)
    batches = [(torch.randn(2, 3, 5, 5, generator=g).contiguous(memory_format=torch.channels_last),
                torch.randint(0, 9, (2,), generator=g)) for _ in range(3)]
    d = _CycleData(batches)
    for t in range(1, 8):
        a = d(t, 0)
        b = d.graph(torch.tensor([t]), 0)
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        assert b[0].is_contiguous(memory_format=torch.channels_last)


def test_schedule_oracle_duration_overrides():
    jobs = [("a", 1, 1, 1, 2), ("b", 1, 1, 1, 2)]
    base, mk = osched.crossover(jobs)
    same, mk2 = osched.crossover(jobs, {})
    assert base == same and mk == mk2 == 9
    # a slower first sync of job a delays a's second compute (Alg. 1), nothing else before it
    slow, mk3 = osched.crossover(jobs, {("a", "sync", 1): 5})
    get = {(s[1], s[2], s[3]): s for s in slow}
    assert get[("a", "sync", 1)][4:] == (2, 7)
    assert get[("a", "forward", 2)][4] == 7 and mk3 > mk
    seq, _ = osched.sequential(jobs, {("b", "backward", 1): 3})
    g2 = {(s[1], s[2], s[3]): s for s in seq}
    assert g2[("b", "sync", 1)][4] == g2[("b", "backward", 1)][5]
    assert np.isclose(g2[("a", "forward", 2)][4], g2[("b", "sync", 1)][5])
