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


def test_bench_self_launch_two_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run
    with 2 ranks (the driver's own N>1 launch line); --dry-run runs the same launch path,
    sharding and max-over-ranks reduction on CPU (gloo) and rank 0 prints one line."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for workload in ("c3", "c5"):
        r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                            "--warmup", "1", "--workload", workload], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
        assert len(lines) == 1, r.stdout
        line = lines[0]
        assert line["n_gpus"] == 2 and line["dry_run"] and line["value"] > 0
        if workload == "c5":
            assert line["shard_rank0"] == list(range(0, 64, 2))  # stream s on GPU s mod 2


def test_bench_config_dicts_match_between_arms():
    """Both arms print the same `config` dict (the driver compares them)."""
    args = bench.parse(["--steps", "1"])
    a = bench.workload_config(args, 1)
    b = bench.workload_config(bench.parse(["--impl", "reference"]), 1)
    assert a == b
