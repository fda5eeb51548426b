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


def _verify_worker(rank, ws, port, q):
    """bench.py's verification plumbing on gloo: each rank computes a deterministic per-row
    function of ITS C2 shard (rows [r*B, (r+1)*B) of the block-seeded global batch), the
    shards are all-gathered to rank 0 and compared bitwise with the same function of the
    whole batch; a tampered shard must be caught."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    from paper_2204_03643_b200 import workloads
    B, n = 1500, 64                       # not a multiple of the 1024-row seeding block

    def f(y, lam):                        # any deterministic row-wise map stands in for the solver
        x = torch.cumsum(torch.as_tensor(y, dtype=torch.float64), dim=1) * torch.as_tensor(lam)[:, None]
        return {"x": x.float(), "mask": (x > 0).to(torch.int32), "lam": torch.as_tensor(lam, dtype=torch.float32)}

    w = workloads.c2(batch=B, n=n, row_offset=rank * B)
    local = f(w.y, w.lam)
    res = {}
    g = bench.gather_to_rank0(local, ws, rank)
    if rank == 0:
        full = workloads.c2(batch=B * ws, n=n)
        res["ok"] = bench.bitwise_compare(g, f(full.y, full.lam), tolerant=("lam",))
    bad = dict(local)
    if rank == 1:
        bad["x"] = bad["x"].clone()
        bad["x"][7, 3] = torch.nextafter(bad["x"][7, 3], torch.tensor(1e9))
    g2 = bench.gather_to_rank0(bad, ws, rank)
    if rank == 0:
        res["bad"] = bench.bitwise_compare(g2, f(full.y, full.lam))
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_verify():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_verify_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ok, bad = res[0]["ok"], res[0]["bad"]
    assert ok["x"] is True and ok["mask"] is True
    assert ok["lam"]["max_abs_diff"] == 0.0
    assert bad["x"] is False and bad["mask"] is True


def test_gpus_flag_mismatch_is_an_error():
    """bench.py --gpus N under a launcher whose WORLD_SIZE differs must refuse to run."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert p.returncode != 0 and "WORLD_SIZE=2" in p.stderr
