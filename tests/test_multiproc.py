"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel plumbing bench.py
uses on B200s: disjoint, covering shards of independent units, per-image seeding that
makes a rank's shard equal to the slice of the full batch, and the max-over-ranks
timing reduction.  The hot path has no data exchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    from paper_2204_03643_b200 import workloads
    total = 7
    off, cnt = bench.shard(total, ws, rank)
    owned = torch.zeros(total, dtype=torch.int64)
    owned[off:off + cnt] = 1
    dist.all_reduce(owned)
    w = workloads.c5(N=cnt, C=3, H=16, W=12, with_grad=True, image_offset=off)
    full = workloads.c5(N=total, C=3, H=16, W=12, with_grad=True)
    same = np.array_equal(w.X, full.X[off:off + cnt]) and np.array_equal(w.grad, full.grad[off:off + cnt])
    t = bench.allreduce_max(float(rank + 1) * 1.5, ws, device="cpu")
    q.put((rank, owned.tolist(), same, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, owned, same, t in res:
        assert owned == [1] * 7          # every unit owned exactly once
        assert same                      # shard == slice of the full seeded batch
        assert t == 3.0                  # max over ranks


def test_shard_edges():
    import bench
    for total in (0, 1, 5, 256):
        for ws in (1, 2, 3, 8):
            got = [bench.shard(total, ws, r) for r in range(ws)]
            assert sum(c for _, c in got) == total
            pos = 0
            for off, c in got:
                assert off == pos
                pos += c
