"""Multi-GPU host logic on CPU: world_size-2 gloo process group (127.0.0.1), the
max-over-ranks timing reduction and the stream / epoch sharding used by bench.py.
The data path has no collective: shards are independent."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", init_method="env://")
    t = bench.max_over_ranks(10.0 + rank, world)
    mine = bench.streams_for_rank(64, world, rank)
    bench.barrier(world)
    q.put((rank, t, mine, bench.epoch_seed(0, rank)))
    dist.destroy_process_group()


def test_two_rank_gloo_reduction_and_sharding():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == 11.0 for r in res)  # max over ranks
    shards = [set(r[2]) for r in res]
    assert shards[0].isdisjoint(shards[1]) and shards[0] | shards[1] == set(range(64))
    assert res[0][3] != res[1][3]  # every rank decodes its own epochs (weak scaling)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_stream_partition_is_complete(world):
    parts = [bench.streams_for_rank(64, world, r) for r in range(world)]
    assert sorted(sum(parts, [])) == list(range(64))
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
