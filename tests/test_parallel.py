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


def test_bench_self_launch_plumbing_gloo():
    """`bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run with 2 ranks; --plumbing-check runs the multi-rank host
    path (head sharding, per-head-seeded inputs, one digest gather, comparison
    with a single-rank recomputation of all heads, max-over-ranks timing) under
    gloo with an input digest in place of the GPU kernels."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--plumbing-check"], capture_output=True, text=True, timeout=300,
                         env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = lines[0]
    assert rec["n_ranks"] == 2 and rec["max_over_ranks"] == 2.0
    assert rec["shards"] == [[0, 3], [3, 3]]
    assert rec["validation"]["heads"] == 6
    assert rec["validation"]["bitwise_equal_to_1gpu_run"] is True


def test_digest_gather_uneven_shards_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_digest_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, g = q.get(timeout=120)
        res[r] = g
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] is None
    assert res[0] == [[float(h), 2.0 * h] for h in range(5)]


def _digest_worker(rank, world, port, q):
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, count = parallel.shard_heads(5, world, rank)
        dig = torch.tensor([[float(h), 2.0 * h] for h in range(start, start + count)],
                           dtype=torch.float64)
        g = bench.gather_digests(dig, 5, world, rank)
        q.put((rank, None if g is None else g.tolist()))
    finally:
        dist.destroy_process_group()
