"""Multi-rank harness path of bench.py on CPU (gloo, world_size 2): every rank searches its own
query shard (weak scaling, no data-path collective) and the job time is the max over ranks."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = bench.shard_queries(1000, rank, world)
        ms = bench.reduce_max_ms(10.0 + 5.0 * rank, world)   # rank 1 is the slow one
        q.put((rank, lo, hi, ms))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_and_max_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shards: same size per rank, disjoint, contiguous
    assert [(lo, hi) for _, lo, hi, _ in got] == [(0, 1000), (1000, 2000)]
    # every rank sees the slowest rank's time
    assert all(ms == 15.0 for *_, ms in got)


def test_single_rank_is_identity():
    assert bench.shard_queries(10_000, 0, 1) == (0, 10_000)
    assert bench.reduce_max_ms(3.5, 1) == 3.5
    assert torch.tensor(1.0).item() == 1.0
