"""Multi-rank host logic of the peer-memory transports on CPU (gloo, world 2 and 3).

Drives the product's own classes -- no GPU needed:
* PeerGroup: the NCCL-free rank group of the p2p / ce transports (no collectives: the NCCL-only
  sync modes are refused with ConfigError);
* the adaptive transport's cross-rank decision (_TransportTuner.decide): ranks that measured
  different rotation periods still keep the SAME transport (sums over the ranks), which the
  peer transports require (a rank on ce and a rank on p2p would not exchange the same data);
* FlagArray's shared-memory rendezvous and its collective failure agreement: rank 0 creates the
  segment, every rank attaches by name; where the page-locking step fails (no CUDA here) every
  rank raises ConfigError together and the segment is unlinked -- no rank is left waiting;
* the nvls transport's multicast-handle passing (a POSIX file descriptor from rank 0 to every rank
  over a UNIX-domain socket).
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_07974_b200.comm import PeerGroup
    from paper_2103_07974_b200.errors import ConfigError
    from paper_2103_07974_b200.p2p import FlagArray, all_ranks_agree
    from paper_2103_07974_b200.scheduler import _TransportTuner

    out = {"rank": rank}
    g = PeerGroup(rank, world)
    out["group"] = (g.rank, g.world, g.has_collectives, g.active)
    try:
        g.all_reduce_(0, 1, 0)
        out["refused"] = False
    except ConfigError:
        out["refused"] = True
    # rank-dependent measurements: rank 0 finds ce faster, the others p2p
    tuner = _TransportTuner()
    medians = [1.0, 2.0] if rank == 0 else [1.0 + 0.2 * world, 1.0]
    tuner.decide(medians, g)
    out["choice"] = tuner.choice
    out["periods"] = tuner.periods_ms
    out["agree_all"] = all_ranks_agree(True)
    out["agree_one_no"] = all_ranks_agree(rank != world - 1)
    # the nvls transport's handle passing: rank 0's file descriptor reaches every rank (SCM_RIGHTS)
    from paper_2103_07974_b200.nvls import _share_fd

    import tempfile

    fd = -1
    if rank == 0:
        tf = tempfile.TemporaryFile()
        tf.write(b"multicast-handle")
        tf.flush()
        fd = os.dup(tf.fileno())
    got = _share_fd(fd, rank, world)
    out["fd_payload"] = os.pread(got, 64, 0) if got >= 0 else None
    if got >= 0:
        os.close(got)
    names_before = set(os.listdir("/dev/shm")) if os.path.isdir("/dev/shm") else set()
    try:
        FlagArray(rank, world)
        out["flags"] = "created"
    except ConfigError as exc:
        out["flags"] = "refused: " + str(exc)[:80]
    dist.barrier()
    names_after = set(os.listdir("/dev/shm")) if os.path.isdir("/dev/shm") else set()
    out["shm_leaked"] = sorted(n for n in names_after - names_before if n.startswith("psm_"))
    allo = [None] * world
    dist.all_gather_object(allo, out)
    if rank == 0:
        q.put(allo)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_group_tuner_and_flag_rendezvous(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert [r["group"] for r in res] == [(r, world, False, False) for r in range(world)]
    assert all(r["refused"] for r in res)
    # sums over ranks: ce = (1 + (W-1)(1 + 0.2W)) / W, p2p = (2 + (W-1)) / W -> one choice everywhere
    assert len({r["choice"] for r in res}) == 1
    ce = (1.0 + (world - 1) * (1.0 + 0.2 * world)) / world
    p2p = (2.0 + (world - 1)) / world
    assert res[0]["choice"] == ("ce" if ce <= p2p else "p2p")
    assert all(abs(r["periods"]["ce"] - ce) < 1e-12 and abs(r["periods"]["p2p"] - p2p) < 1e-12 for r in res)
    assert all(r["agree_all"] for r in res) and not any(r["agree_one_no"] for r in res)
    assert all(r["fd_payload"] == b"multicast-handle" for r in res)
    # without CUDA page-locking fails on every rank, and every rank refuses together
    import torch

    want = "created" if torch.cuda.is_available() else "refused"
    assert all(r["flags"].startswith(want) for r in res), res
    assert all(not r["shm_leaked"] for r in res)


def test_gather_chunks_cover_every_shard_exactly_once():
    """The p2p_gather work list (fusion.gather_chunks): over the W shards of a padded, sharded
    bucket layout (ResNet-50's 161 tensors and a ragged set), every gradient element is covered by
    exactly one chunk, no chunk crosses a tensor or a shard, chunks hold at most `ch` elements and
    start 16-byte aligned inside their tensor (the kernel's vector path), padding is never touched."""
    import numpy as np

    from paper_2103_07974_b200.fusion import gather_chunks
    from paper_2103_07974_b200.workload import BucketLayout

    rng = np.random.default_rng(0)
    sizes = [[int(x) for x in rng.integers(1, 70000, 40)] + [10, 3, 256 * 784, 1],
             [64 * 3 * 7 * 7, 64, 64, 64 * 64, 64, 64, 2048 * 1000, 1000]]
    for numels in sizes:
        for world in (2, 3, 4, 8):
            lay = BucketLayout.build(numels, 32, multiple=32 * world)
            shard = lay.total // world
            ch = {2: 4096, 3: 2048, 4: 2048}.get(world, 1024)
            seen = np.zeros(lay.total, dtype=np.int32)
            for r in range(world):
                s0, s1 = r * shard, (r + 1) * shard
                for i, o, a, b in gather_chunks(lay.offsets, lay.numels, s0, s1, ch):
                    assert o == lay.offsets[i] and o <= a < b <= o + lay.numels[i]
                    assert s0 <= a and b <= s1 and b - a <= ch and (a - o) % 4 == 0
                    seen[a:b] += 1
            want = np.zeros(lay.total, dtype=np.int32)
            for o, n in zip(lay.offsets, lay.numels):
                want[o:o + n] = 1
            assert np.array_equal(seen, want)
