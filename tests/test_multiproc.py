"""Host-side logic of the multi-GPU (replica) bench path, run with world_size 2 over gloo on CPU.

bench.py --gpus N runs N independent replicas: rank r solves systems r, r+N, ...
of the cfg 3 sequence; timings are reduced with MAX over ranks; value = systems solved by all ranks /
max time.  No data-path collective exists (the path does not shard within a solve).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        systems = [bench.system_of(rank, world, k, 10) for k in range(7)]
        local = 100.0 + 25.0 * rank
        m = bench.max_over_ranks(local, world, None)
        gathered = [None] * world
        dist.all_gather_object(gathered, systems)
        q.put((rank, systems, m, gathered))
    finally:
        dist.destroy_process_group()


def test_replica_schedule_and_max_reduction():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, systems, m, gathered in out:
        assert m == 125.0                           # max over ranks
        assert systems == [(rank + 2 * k) % 10 for k in range(7)]
    # ranks cover disjoint systems in each round; together they cycle through the whole sequence
    s0, s1 = out[0][3]
    assert all(a != b for a, b in zip(s0, s1))
    assert sorted(set(s0[:5] + s1[:5])) == list(range(10))


def test_single_rank_is_identity():
    assert bench.max_over_ranks(3.5, 1) == 3.5
    assert [bench.system_of(0, 1, k, 10) for k in range(12)] == [k % 10 for k in range(12)]
