"""World-size-2 gloo tests of the multi-rank host logic (no GPU needed)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_15180_b200 import parallel


def test_shard_heads_partition():
    for total in (1, 7, 64, 256):
        for n in (1, 2, 4, 8):
            spans = [parallel.shard_heads(total, n, r) for r in range(n)]
            covered = [h for s, c in spans for h in range(s, s + c)]
            assert covered == list(range(total))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        parallel.shard_heads(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assert parallel.world() == (rank, world)
        m = parallel.max_over_ranks(10.0 + rank)
        s = parallel.sum_over_ranks(1.0 + rank)
        start, count = parallel.shard_heads(5, world, rank)
        t = torch.full((count, 3), float(rank))
        pad = torch.zeros(3 - count, 3) if count < 3 else torch.zeros(0, 3)
        g = parallel.gather_to_rank0(torch.cat([t, pad]) if count < 3 else t)
        q.put((rank, m, s, None if g is None else g.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r, m, s, g = q.get(timeout=120)
        out[r] = (m, s, g)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] == out[1][0] == 11.0  # max over ranks
    assert out[0][1] == out[1][1] == 3.0   # sum over ranks
    assert out[1][2] is None
    g = out[0][2]
    assert len(g) == 6 and g[0][0] == 0.0 and g[3][0] == 1.0
