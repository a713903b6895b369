"""N > 1 host path of bench.py on the CPU (gloo, world_size 2): replicas only,
timing reduced as the max over ranks, whole-job value = ranks x bytes / max time, and the
reference arm printing on rank 0 only."""

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
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = [10.0 + rank, 4.0 - rank, 6.0 + 2 * rank]
    got = bench.reduce_max(mine, dist)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, got))


def test_max_over_ranks_with_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == [11.0, 4.0, 8.0]


def test_job_value_is_weak_scaling_aggregate():
    import bench

    assert bench.job_value(1, 4e9, 1000.0) == pytest.approx(4.0)
    assert bench.job_value(8, 4e9, 1000.0) == pytest.approx(32.0)
    assert bench.reduce_max([1, 2], None) == [1.0, 2.0]


def test_reference_arm_prints_on_rank_zero_only(capsys):
    import argparse

    import bench

    args = argparse.Namespace(workload="c1", steps=1, warmup=0, gpus=2)
    bench.run_reference(args, world=2, rank=1)
    assert capsys.readouterr().out == ""
