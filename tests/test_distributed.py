"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): the
max-over-ranks timing, the whole-job sums, and the config-4 trace partition."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    import torch.distributed as dist

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t = bench.max_over_ranks(1.5 + rank, world)
    s = bench.sum_over_ranks(100.0 * (rank + 1), world)
    cells = bench.config4_cells()
    mine = list(range(rank, len(cells), 8))[:128]
    q.put((rank, t, s, mine))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, s0, m0), (r1, t1, s1, m1) = out
    assert t0 == t1 == 2.5          # max over ranks
    assert s0 == s1 == 300.0        # whole-job sum
    assert len(m0) == len(m1) == 128 and not set(m0) & set(m1)


def test_config4_partition_covers_all_cells():
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    cells = bench.config4_cells()
    assert len(cells) == 1024 and len(set(cells)) == 1024
    shares = [list(range(r, 1024, 8))[:128] for r in range(8)]
    assert sorted(i for s in shares for i in s) == list(range(1024))


class _FakeShard:
    """Stands in for Engine(shards=W, shard_rank=r): the host side of the
    mailbox-handle exchange only (no device)."""

    def __init__(self, rank):
        self.rank = rank
        self.got = None

    def mailbox_handle(self):
        return bytes([self.rank + 1]) * 64

    def connect_shards(self, handles):
        self.got = handles


def _shard_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    import torch.distributed as dist

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_11546_b200 import sharded

    eng = _FakeShard(rank)
    sharded.connect(eng)
    q.put((rank, eng.got))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_shard_handle_exchange():
    """Every rank receives every shard's mailbox handle, in rank order (sharded.connect)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([1]) * 64, bytes([2]) * 64]
    assert out[0][1] == want and out[1][1] == want


def test_shard_head_merge_equals_global_order():
    """The sharded waiting head (min over shards of each shard's min (priority bits,
    rank) over the relQueries it owns, a % W) is the unsharded head, ties included."""
    import numpy as np

    rng = np.random.default_rng(7)
    for W in (2, 3, 8):
        for _ in range(200):
            R = int(rng.integers(1, 300))
            prio = rng.choice([0.0, 0.5, 1.25, 3.0], size=R) if rng.random() < 0.5 else rng.random(R)
            waiting = rng.random(R) < 0.7
            bits = prio.view(np.uint64)
            keys = [(int(bits[a]), a) for a in range(R) if waiting[a]]
            want = min(keys) if keys else None
            heads = []
            for s in range(W):
                own = [k for k in keys if k[1] % W == s]
                if own:
                    heads.append(min(own))
            assert (min(heads) if heads else None) == want
