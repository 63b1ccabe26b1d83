"""The N>1 path of bench.py (replicas only) on CPU with the
gloo backend, world_size 2: barrier, max/sum over ranks and the whole-job
throughput formula."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as td
    import bench
    td.init_process_group("gloo", rank=rank, world_size=world)
    bench.barrier(td)
    mx = bench.max_over_ranks(td, 1.0 + rank)
    sm = bench.sum_over_ranks(td, 10.0)
    # rank r times 2.0 + r ms per step over 5 steps of 1 GB
    v, t = bench.replica_throughput(td, 1e9, 5, 2.0 + rank)
    q.put((rank, mx, sm, v, t))
    td.destroy_process_group()


def test_replicas_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, sm, v, t in res:
        assert mx == 2.0 and sm == 20.0
        assert t == 3.0                                  # slowest rank defines the time
        assert abs(v - 1e9 * 10 / (3e-3 * 5) / 1e9) < 1e-9  # all ranks' steps / max time
