#!/usr/bin/env python
"""Benchmark of the batched TV-prox hot path on B200 (arXiv 2204.03643).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--verify|--no-verify]

`--gpus N > 1` re-launches itself under `torch.distributed.run` (one rank per GPU,
NCCL, 127.0.0.1) unless it already runs under torchrun, in which case WORLD_SIZE must
equal N.

Headline (`value`): BASELINE.json configs[1] = C2, batched 1D TV prox fwd+bwd, 65536
rows x 1024 samples per GPU, per-row lambda, fp32 -> rows/s over all ranks.  A step =
one forward (projected-Newton prox + saved mask) and one backward (segment-mean VJP +
per-row lambda gradient) over the batch; inputs resident in HBM; every tensor (256 MiB)
exceeds L2 (126 MB).  Weak scaling: rank r owns rows [r*65536, (r+1)*65536) of one
seeded global batch; no collective on the data path (rows are independent problems),
NCCL only for the barrier, the max-over-ranks timing reduction and the verification.

`configs`: every BASELINE config and Table 1's two shapes, fwd and bwd timed
separately with an L2 flush (256 MiB write) before each timed call: C1 and T1a/T1b
(1D, replicated per rank), C3 / C4 / C5 (2D, images sharded over ranks, strong
scaling), the 2D ones also replayed as CUDA graphs; per-pass PN iteration mean / p99 /
max from the per-call iteration histogram; R1 (whole-op) HBM roofline per config.
`e2e`: the C2 metric through the public API with pinned host buffers, H2D of
y/lambda/grad_x and D2H of x/grad_y/grad_lambda inside the timed region, every rank.
`verify` (outside the timed region): outputs all-gathered to rank 0 over NCCL and
compared BITWISE with rank 0's own single-GPU solve of the whole global batch, plus
an oracle check of sampled rows / planes.
`cpu_baseline`: the CPU oracle (oracle/, fp64 C) on bounded samples of C2 and C5 on
the host cores (rank 0, N = 1 only), with a single-thread number and the CPU model.
`--impl reference`: the oracle timed as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2_ROWS, C2_N = 65536, 1024
METRIC = "TV-prox fwd+bwd rows/sec (1D C2) ; 2D Mpixel/sec (C5) ; % HBM roofline"
WORKLOAD = "C2: batched 1D TV prox fwd+bwd, 65536 x 1024 per GPU, per-row lambda, fp32 (BASELINE.json configs[1])"
FLUSH_BYTES = 256 << 20         # > 2 x the 126 MB L2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


def load_profile_json(name):
    """Per-launch ncu numbers from the committed captures (profiles/<name>), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return {}


REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                bits = int(parts[2], 16)
                for b, name in REASON_BITS.items():
                    if bits & b and name != "gpu_idle":
                        reasons.add(name)
            except ValueError:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- distributed plumbing
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(n):
    """`bench.py --gpus N` outside torchrun: re-exec as N ranks (one per GPU) and return
    the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup(backend="nccl"):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def shard(total, ws, rank):
    """Contiguous block of `total` independent units (images / rows) owned by `rank`."""
    base, rem = divmod(total, ws)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def allreduce_max(x, ws, device="cuda"):
    """Max over ranks (the timing rule: the slowest rank sets the step time)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    import torch
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def gather_to_rank0(local, ws, rank):
    """All-gather each tensor of `local` (same shape on every rank, contiguous blocks of one
    global batch in rank order) and return the concatenations on rank 0 (None elsewhere).
    NCCL for CUDA tensors, gloo for CPU tensors (tests/test_multiproc.py)."""
    import torch
    if ws == 1:
        return dict(local)
    import torch.distributed as dist
    out = {}
    for name, t in local.items():
        t = t.contiguous()
        parts = [torch.empty_like(t) for _ in range(ws)]
        dist.all_gather(parts, t)
        out[name] = torch.cat(parts) if rank == 0 else None
    return out if rank == 0 else None


def bitwise_compare(gathered, reference, tolerant=()):
    """Per tensor: bitwise equality of the gathered N-rank result with the single-device
    reference (the library's determinism contract, include/tvprox.h), except names in
    `tolerant` (cross-rank partial sums), which report the max relative difference."""
    import torch
    res = {}
    for name, ref in reference.items():
        g = gathered[name]
        if name in tolerant:
            d = (g.double() - ref.double()).abs().max().item()
            res[name] = {"max_abs_diff": d, "rel": d / max(ref.double().abs().max().item(), 1e-30)}
        else:
            res[name] = bool(g.shape == ref.shape and torch.equal(g.view(torch.uint8) if g.dtype != torch.uint8 else g,
                                                                ref.view(torch.uint8) if ref.dtype != torch.uint8
                                                                else ref))
    return res


# --------------------------------------------------------------------------- timing helpers
class Flusher:
    def __init__(self, dev):
        import torch
        self.buf = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def __call__(self):
        self.buf.zero_()


def ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def stats_ms(v):
    return {"mean": statistics.mean(v), "median": statistics.median(v),
            "std": statistics.pstdev(v) if len(v) > 1 else 0.0, "reps": len(v)}


def iter_stats(hist_row):
    """mean / p99 / max PN iterations of one pass from its iteration histogram."""
    h = np.asarray(hist_row, np.int64)
    tot = int(h.sum())
    if tot == 0:
        return None
    bins = np.arange(h.size)
    conv = h[:-1]
    c = np.cumsum(conv)
    p99 = int(np.searchsorted(c, 0.99 * conv.sum())) if conv.sum() else 0
    nz = np.nonzero(conv)[0]
    return {"mean": float((bins[:-1] * conv).sum() / max(conv.sum(), 1)), "p99": p99,
            "max": int(nz.max()) if nz.size else 0, "not_converged": int(h[-1]), "lines": tot}


# --------------------------------------------------------------------------- ours: C2 headline
def bench_c2(args, ws, rank, local):
    import torch
    from paper_2204_03643_b200 import _lib, tvprox, workloads
    lib = _lib.load()
    w = workloads.c2(batch=C2_ROWS, row_offset=rank * C2_ROWS)
    dev = torch.device("cuda", local)
    y = torch.as_tensor(w.y, device=dev)
    lam = torch.as_tensor(w.lam.astype(np.float32), device=dev)
    g = torch.as_tensor(w.grad, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(evs=None):
        if evs is not None:
            evs[0].record(stream)
        x, mask, _ = tvprox.tv1d_fwd(y, lam, need_mask=True)
        if evs is not None:
            evs[1].record(stream)
        gy, gl = tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW, want_lam=True)
        if evs is not None:
            evs[2].record(stream)
        return x, gy, gl

    evs = [[ev() for _ in range(3)] for _ in range(args.steps)]
    clk = ClockSampler(local)
    clk.start()
    time.sleep(1.0)          # let nvidia-smi finish its NVML start-up before the timed region
    # warm-up right before the timed region (outputs held across steps exactly as in the
    # timed loop, so the caching allocator owns every block before timing starts)
    out = None
    for _ in range(args.warmup):
        out = step()
    lib.tvp_launch_count(1)
    barrier(ws)
    t0, t1 = ev(), ev()
    t0.record(stream)
    for i in range(args.steps):
        out = step(evs[i])
    t1.record(stream)
    barrier(ws)
    launches = lib.tvp_launch_count(1)
    clocks = clk.stop()
    ms = t0.elapsed_time(t1)
    fwd_ms = [e[0].elapsed_time(e[1]) for e in evs]
    bwd_ms = [e[1].elapsed_time(e[2]) for e in evs]
    print("[bench] rank %d per-step fwd ms: %s" % (rank, " ".join("%.3f" % v for v in fwd_ms)), file=sys.stderr)
    print("[bench] rank %d per-step bwd ms: %s" % (rank, " ".join("%.3f" % v for v in bwd_ms)), file=sys.stderr)
    ms_max = allreduce_max(ms, ws)
    # iteration statistics (outside the timed region)
    hist = torch.zeros((1, _lib.HIST_BINS), dtype=torch.int32, device=dev)
    diag = torch.zeros(4, dtype=torch.int32, device=dev)
    _, _, it = tvprox.tv1d_fwd(y, lam, need_mask=True, want_iters=True,
                               opts=tvprox.make_options(diag=diag, iter_hist=hist))
    itn = it.cpu().numpy()
    res = {
        "ms": ms_max, "ms_local": ms, "fwd_ms": allreduce_max(statistics.mean(fwd_ms), ws),
        "bwd_ms": allreduce_max(statistics.mean(bwd_ms), ws),
        "fwd_ms_median": statistics.median(fwd_ms), "bwd_ms_median": statistics.median(bwd_ms),
        "launches": launches, "clocks": clocks,
        "iters": dict(iter_stats(hist[0].cpu().numpy()),
                      stall_accepts=int(((itn >= 0) & ((itn >> 16) & 1 == 1)).sum()),
                      line_search_rows=int(diag[1].item())),
        "host": (w.y, w.lam.astype(np.float32), w.grad),
        "dev": (y, lam, g), "out": out,
    }
    return res


def bench_c2_e2e(args, host, ws, local, chunks=8):
    """Public-API end-to-end on every rank: pinned host -> device, fwd+bwd, device -> pinned
    host, every step.  The rank's batch is streamed in `chunks` row blocks over two CUDA
    streams, so the H2D copy of block i+1, the kernels of block i and the D2H copy of block
    i-1 overlap (rows are independent problems; PCIe is full duplex).  Every byte of every
    step's inputs and results still crosses the bus inside the timed region."""
    import torch
    from paper_2204_03643_b200 import _lib, tvprox
    dev = torch.device("cuda", local)
    y_h = torch.from_numpy(host[0]).pin_memory()
    l_h = torch.from_numpy(host[1]).pin_memory()
    g_h = torch.from_numpy(host[2]).pin_memory()
    x_o = torch.empty_like(y_h).pin_memory()
    gy_o = torch.empty_like(g_h).pin_memory()
    gl_o = torch.empty_like(l_h).pin_memory()
    rows = y_h.shape[0]
    bounds = [(rows * c // chunks, rows * (c + 1) // chunks) for c in range(chunks)]
    streams = [torch.cuda.Stream(dev) for _ in range(2)]
    main = torch.cuda.current_stream(dev)

    def step():
        for s in streams:
            s.wait_stream(main)
        for c, (a, b) in enumerate(bounds):
            s = streams[c % 2]
            with torch.cuda.stream(s):
                y = y_h[a:b].to(dev, non_blocking=True)
                lam = l_h[a:b].to(dev, non_blocking=True)
                g = g_h[a:b].to(dev, non_blocking=True)
                x, mask, _ = tvprox.tv1d_fwd(y, lam, need_mask=True)
                gy, gl = tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW, want_lam=True)
                x_o[a:b].copy_(x, non_blocking=True)
                gy_o[a:b].copy_(gy, non_blocking=True)
                gl_o[a:b].copy_(gl, non_blocking=True)
        for s in streams:
            main.wait_stream(s)

    for _ in range(2):
        step()
    barrier(ws)
    k = max(2, min(args.steps, 8))
    t0, t1 = ev(), ev()
    t0.record(main)
    for _ in range(k):
        step()
    t1.record(main)
    barrier(ws)
    ms = allreduce_max(t0.elapsed_time(t1) / k, ws)
    h2d = y_h.numel() * 4 + l_h.numel() * 4 + g_h.numel() * 4
    d2h = x_o.numel() * 4 + gy_o.numel() * 4 + gl_o.numel() * 4
    return ms, h2d, d2h


# --------------------------------------------------------------------------- ours: per-config lines
def _bytes_1d(rows, n, itemsize):
    """Algorithmic bytes of a 1D fwd or bwd over `rows` rows: read n, write n, the 2-bit
    mask, one lambda (fwd) / one lambda gradient (bwd) per row."""
    return rows * (2 * n * itemsize + 4 * ((n - 2) // 16 + 1 if n > 1 else 0) + itemsize)


def _bytes_2d(planes, H, W, K, itemsize):
    """R1 (whole-op) algorithmic bytes of a 2D fwd or bwd: read the input plane, write the
    output plane, write (fwd) / read (bwd) the 2K saved masks."""
    mw = lambda n: (n - 2) // 16 + 1 if n > 1 else 0  # noqa: E731
    return planes * (2 * H * W * itemsize + K * (H * mw(W) + W * mw(H)) * 4)


def time_1d_config(w, dev, ws, reps, flush, peak):
    """1D config timed like the paper's Table 1 protocol (mean +- std of reps runs), fwd and
    bwd separately, L2 flushed before each timed call."""
    import torch
    from paper_2204_03643_b200 import _lib, tvprox
    dt = torch.float64 if w.dtype == "f64" else torch.float32
    y = torch.as_tensor(w.y, dtype=dt, device=dev)
    g = torch.as_tensor(w.grad, dtype=dt, device=dev)
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam, dtype=dt, device=dev)
    mode = {"scalar": _lib.LAM_SCALAR, "row": _lib.LAM_PER_ROW}[w.lam_mode]
    for _ in range(3):
        x, mask, _ = tvprox.tv1d_fwd(y, lam)
        tvprox.tv1d_bwd(g, mask, mode)
    f, b = [], []
    for _ in range(reps):
        e = [ev() for _ in range(4)]
        flush()
        e[0].record()
        x, mask, _ = tvprox.tv1d_fwd(y, lam)
        e[1].record()
        flush()
        e[2].record()
        tvprox.tv1d_bwd(g, mask, mode)
        e[3].record()
        torch.cuda.synchronize()
        f.append(e[0].elapsed_time(e[1]))
        b.append(e[2].elapsed_time(e[3]))
    hist = torch.zeros((1, _lib.HIST_BINS), dtype=torch.int32, device=dev)
    tvprox.tv1d_fwd(y, lam, opts=tvprox.make_options(iter_hist=hist))
    rows, n = w.y.shape
    fm, bm = allreduce_max(statistics.mean(f), ws), allreduce_max(statistics.mean(b), ws)
    nb = _bytes_1d(rows, n, 8 if w.dtype == "f64" else 4)
    return {"shape": [rows, n], "dtype": w.dtype, "lam": w.lam_mode, "fwd_ms": stats_ms(f), "bwd_ms": stats_ms(b),
            "value": rows * ws / ((fm + bm) * 1e-3), "unit": "rows/s (fwd+bwd, all ranks)",
            "r1_frac": {"fwd": nb / (fm * 1e-3) / 1e9 / peak, "bwd": nb / (bm * 1e-3) / 1e9 / peak},
            "pn_iters": iter_stats(hist[0].cpu().numpy()), "l2": "flushed before each timed call",
            "scaling": "weak (replicated per rank)"}


def time_2d_config(w, dev, ws, reps, flush, peak, graph=True, cluster=False):
    """2D config: fwd (training, saved masks) and bwd (with lambda gradient) timed
    separately with an L2 flush before each, eager and as CUDA graphs; per-pass PN
    iteration statistics from the iteration histogram."""
    import torch
    from paper_2204_03643_b200 import _lib, tvprox
    X = torch.as_tensor(w.X, device=dev)
    G = torch.as_tensor(w.grad, device=dev)
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam.astype(np.float32), device=dev)
    mode = {"scalar": _lib.LAM_SCALAR, "channel": _lib.LAM_PER_CHANNEL, "plane": _lib.LAM_PER_PLANE}[w.lam_mode]
    K = w.iters

    def fwd():
        return tvprox.tv2d_fwd(X, lam, K, training=True)

    def bwd(saved):
        return tvprox.tv2d_bwd(G, saved, mode, K, want_lam=True)

    for _ in range(3):
        Y, saved, _ = fwd()
        bwd(saved)
    torch.cuda.synchronize()

    def run(ffn, bfn):
        f, b = [], []
        for _ in range(reps):
            e = [ev() for _ in range(4)]
            flush()
            e[0].record()
            s = ffn()
            e[1].record()
            flush()
            e[2].record()
            bfn(s)
            e[3].record()
            torch.cuda.synchronize()
            f.append(e[0].elapsed_time(e[1]))
            b.append(e[2].elapsed_time(e[3]))
        return f, b

    f, b = run(lambda: fwd()[1], bwd)
    out = {}
    if graph:
        gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf):
            Yg, sg, _ = fwd()
        with torch.cuda.graph(gb):
            GXg, glg = bwd(sg)
        gfm, gbm = run(lambda: gf.replay(), lambda s: gb.replay())
        out["graph"] = {"fwd_ms": stats_ms(gfm), "bwd_ms": stats_ms(gbm)}
    if cluster:
        # f2 on a thread-block cluster (tvp_options_t.fused2d = 1): on-chip plane state, bitwise
        # the same result; reported beside the default (staged) path it is measured against
        oc = tvprox.make_options(fused2d=1)
        Yc, sc, _ = tvprox.tv2d_fwd(X, lam, K, training=True, opts=oc)
        cf, cb = run(lambda: tvprox.tv2d_fwd(X, lam, K, training=True, opts=oc)[1],
                     lambda s: tvprox.tv2d_bwd(G, s, mode, K, want_lam=True, opts=oc))
        out["cluster_f2"] = {"fwd_ms": stats_ms(cf), "bwd_ms": stats_ms(cb),
                             "bitwise_equal_to_default": bool(torch.equal(Yc, Y) and torch.equal(sc, saved))}
    hist = torch.zeros((2 * K, _lib.HIST_BINS), dtype=torch.int32, device=dev)
    tvprox.tv2d_fwd(X, lam, K, training=False, opts=tvprox.make_options(iter_hist=hist))
    hn = hist.cpu().numpy()
    N, C, H, W = w.X.shape
    fm, bm = allreduce_max(statistics.mean(f), ws), allreduce_max(statistics.mean(b), ws)
    px = N * C * H * W
    nb = _bytes_2d(N * C, H, W, K, 4)
    out.update({
        "shape_per_rank": [N, C, H, W], "K": K, "lam": w.lam_mode, "fwd_ms": stats_ms(f), "bwd_ms": stats_ms(b),
        "value": px * ws / ((fm + bm) * 1e-3) / 1e6, "unit": "Mpixel/s (NCHW elements, fwd+bwd, all ranks)",
        "spatial_mpx_per_s": px * ws / C / ((fm + bm) * 1e-3) / 1e6,
        "r1_frac": {"fwd": nb / (fm * 1e-3) / 1e9 / peak, "bwd": nb / (bm * 1e-3) / 1e9 / peak},
        "algorithmic_bytes_per_rank": {"fwd": nb, "bwd": nb},
        "pn_iters_per_pass": [dict(iter_stats(hn[p]), name="%s%d" % ("row" if p % 2 == 0 else "col", p // 2 + 1))
                              for p in range(2 * K)],
        "l2": "flushed before each timed call", "scaling": "strong (images sharded over ranks)",
    })
    return out


def bench_configs(args, ws, rank, local, peak):
    import torch
    from paper_2204_03643_b200 import workloads
    dev = torch.device("cuda", local)
    flush = Flusher(dev)
    res = {}
    reps = 25                     # the paper's 25 runs
    res["C1"] = time_1d_config(workloads.c1(), dev, ws, reps, flush, peak)
    res["T1a"] = time_1d_config(workloads.t1("a"), dev, ws, reps, flush, peak)
    res["T1b"] = time_1d_config(workloads.t1("b"), dev, ws, reps, flush, peak)
    # f4: long 1D signals -- one CTA per row up to 8192 samples, a thread-block cluster beyond
    for n in (8192, 16384, 65536):
        res["L%d" % n] = time_1d_config(workloads.long_rows(n), dev, ws, 5, flush, peak)
    barrier(ws)
    for name, fn, total in (("C3", workloads.c3, 64), ("C4", workloads.c4, 16), ("C5", workloads.c5, 256)):
        off, per = shard(total, ws, rank)
        if name == "C5":
            w = fn(N=per, image_offset=off)
        else:
            w = fn()
            w.X = np.ascontiguousarray(w.X[off:off + per])
            w.grad = np.ascontiguousarray(w.grad[off:off + per])
        barrier(ws)
        res[name] = time_2d_config(w, dev, ws, 10 if name == "C5" else 20, flush, peak, cluster=name == "C5")
        res[name]["images_per_rank"] = per
        del w
        torch.cuda.empty_cache()
    return res


# --------------------------------------------------------------------------- ours: verification
def verify(c2, ws, rank, local, with_c5=True):
    """Outside the timed region.  C2: every rank's (x, grad_y, grad_lambda) all-gathered to
    rank 0 and compared bitwise with rank 0's single-GPU solve of the whole global batch;
    oracle parity of 64 sampled rows.  C5: 2D outputs of the sharded images gathered and
    compared bitwise with a single-GPU solve of all of them (lambda gradients: cross-rank
    partial sums, compared within tolerance)."""
    import torch
    import oracle
    from paper_2204_03643_b200 import _lib, tvprox, workloads
    dev = torch.device("cuda", local)
    x, gy, gl = c2["out"]
    gathered = gather_to_rank0({"x": x, "grad_y": gy, "grad_lam": gl}, ws, rank)
    res = {"ranks": ws}
    if rank == 0:
        full = workloads.c2(batch=C2_ROWS * ws)
        y = torch.as_tensor(full.y, device=dev)
        lam = torch.as_tensor(full.lam.astype(np.float32), device=dev)
        g = torch.as_tensor(full.grad, device=dev)
        xr, mask, _ = tvprox.tv1d_fwd(y, lam)
        gyr, glr = tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW)
        res["c2_bitwise_vs_single_gpu"] = bitwise_compare(gathered, {"x": xr, "grad_y": gyr, "grad_lam": glr})
        pick = np.sort(np.random.default_rng(7).choice(C2_ROWS * ws, 64, replace=False))
        xo, brk, sgn = oracle.prox1d_batch(full.y[pick].astype(np.float64), full.lam[pick], nthreads=8)
        xg = gathered["x"][torch.as_tensor(pick, device=dev)].double().cpu().numpy()
        rngy = float(np.ptp(full.y[pick]))
        res["c2_oracle_sample"] = {"rows": 64, "max_err_rel_range": float(np.abs(xg - xo).max() / rngy),
                                   "tol": 1e-4}
        del y, g, xr, gyr, mask
    if with_c5:
        off, per = shard(256, ws, rank)
        w = workloads.c5(N=per, image_offset=off)
        X = torch.as_tensor(w.X, device=dev)
        lamc = torch.as_tensor(w.lam.astype(np.float32), device=dev)
        Y, saved, _ = tvprox.tv2d_fwd(X, lamc, 4)
        GX, gl5 = tvprox.tv2d_bwd(torch.as_tensor(w.grad, device=dev), saved, _lib.LAM_PER_CHANNEL, 4)
        if ws > 1:
            import torch.distributed as dist
            dist.all_reduce(gl5)                   # per-rank partial sums (include/tvprox.h)
        g5 = gather_to_rank0({"Y": Y, "grad_X": GX}, ws, rank)
        if rank == 0:
            w1 = w if ws == 1 else workloads.c5(N=256)
            X1 = torch.as_tensor(w1.X, device=dev)
            Y1, s1, _ = tvprox.tv2d_fwd(X1, lamc, 4)
            GX1, gl1 = tvprox.tv2d_bwd(torch.as_tensor(w1.grad, device=dev), s1, _lib.LAM_PER_CHANNEL, 4)
            g5["grad_lam"] = gl5
            res["c5_bitwise_vs_single_gpu"] = bitwise_compare(g5, {"Y": Y1, "grad_X": GX1, "grad_lam": gl1},
                                                              tolerant=("grad_lam",))
            p = [0, 400, 767]
            Yo, _ = oracle.prox2d_batch(w1.X.reshape(768, 224, 224)[p].astype(np.float64),
                                        np.tile(w1.lam, 256)[p], 4, nthreads=3)
            Yg = g5["Y"].reshape(768, 224, 224)[p].double().cpu().numpy()
            res["c5_oracle_sample"] = {"planes": p, "max_err_rel_range": float(np.abs(Yg - Yo).max() / np.ptp(w1.X)),
                                       "tol": 1e-4}
    barrier(ws)
    return res if rank == 0 else None


# --------------------------------------------------------------------------- CPU baseline (oracle)
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(seconds=10.0, rows_per_batch=4096):
    """The oracle as it stands on the host cores: C2 rows fwd (taut string) + bwd (segment
    mean), all cores and one thread; C5 planes (Alg. 1 + reverse mode) on all cores."""
    import oracle
    from paper_2204_03643_b200 import workloads
    cores = os.cpu_count() or 1
    w = workloads.c2(batch=rows_per_batch * 4, with_grad=True)
    oracle.build()

    def run(nthreads, budget, rows):
        done, t_start, b = 0, time.perf_counter(), 0
        while True:
            sl = slice((b % 4) * rows, (b % 4 + 1) * rows)
            x, brk, sgn = oracle.prox1d_batch(w.y[sl].astype(np.float64), w.lam[sl], nthreads=nthreads)
            oracle.bwd1d_batch(brk, sgn, w.grad[sl].astype(np.float64), nthreads=nthreads)
            done += rows
            b += 1
            el = time.perf_counter() - t_start
            if el >= budget:
                return done, el

    done, el = run(cores, seconds, rows_per_batch)
    d1, e1 = run(1, 3.0, 512)
    n5 = 128
    w5 = workloads.c5(N=n5)
    P = 3 * n5
    Xp = w5.X.reshape(P, 224, 224).astype(np.float64)
    G5 = w5.grad.reshape(P, 224, 224).astype(np.float64)
    t0 = time.perf_counter()
    Yr, segs = oracle.prox2d_batch(Xp, np.tile(w5.lam, n5), 4, nthreads=cores)
    oracle.bwd2d_batch(segs, G5, 4, nthreads=cores)
    e5 = time.perf_counter() - t0
    return {"value": done / el, "unit": "rows/s", "cores": cores, "kind": "oracle",
            "sample": "%d C2 rows (1024 samples, per-row lambda) fwd+bwd in %.1f s, fp64 C oracle, %d threads"
                      % (done, el, cores),
            "cpu_model": cpu_model(),
            "single_thread": {"value": d1 / e1, "unit": "rows/s", "cores": 1,
                              "sample": "%d C2 rows fwd+bwd in %.1f s, 1 thread" % (d1, e1)},
            "c5_2d": {"value": P * 224 * 224 / e5 / 1e6, "unit": "Mpixel/s", "cores": cores,
                      "sample": "%d C5 images (%d planes of 224^2, K = 4) fwd + reverse mode in %.1f s" % (n5, P, e5)}}


def issue_roofline(warp_instr, ms, peaks):
    """Instruction-issue roofline of the forward op: executed warp instructions per launch
    (ncu, committed profile) over its live duration, against the SM issue peak
    (148 SMs x 4 schedulers x 1 warp-instruction / clock at the max SM clock)."""
    if not warp_instr or not ms:
        return None
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0)) if peaks else 1965.0
    peak = 148 * 4 * sm_mhz * 1e6
    ach = warp_instr / (ms * 1e-3)
    return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-instr/s", "frac": ach / peak,
            "warp_instr_per_launch": warp_instr, "source": "ncu smsp__inst_executed (profiles/ncu_traffic.json)"}


def run_ours(args):
    import torch
    ws, rank, local = dist_setup()
    peak, peak_src, peaks = load_peaks()
    traffic = load_profile_json("ncu_traffic.json")
    r = bench_c2(args, ws, rank, local)
    rows_total = C2_ROWS * ws
    value = rows_total / (r["ms"] * 1e-3 / args.steps)
    ms_step = r["ms"] / args.steps
    # roofline of the dominant kernel (the forward PN op): algorithmic bytes per launch
    fwd_bytes = _bytes_1d(C2_ROWS, C2_N, 4)
    bwd_bytes = _bytes_1d(C2_ROWS, C2_N, 4)
    fwd_gbs = fwd_bytes / (r["fwd_ms"] * 1e-3) / 1e9
    bwd_gbs = bwd_bytes / (r["bwd_ms"] * 1e-3) / 1e9
    roof = {
        "kernel": "tv1d_prox_fwd = k_coarse_rows4 (coarse bound set) + k_row_fwd_w<float,16,2> (projected "
                  "Newton, 2 warps/line)",
        "bound": "hbm", "achieved": fwd_gbs, "peak": peak, "unit": "GB/s", "frac": fwd_gbs / peak,
        "peak_source": peak_src,
        # DRAM bytes of ALL kernels of the op (coarse pre-pass + fine solve), ncu --set full
        "traffic": traffic.get("c2_fwd_op_bytes_per_launch", traffic.get("c2_fwd_bytes_per_launch")),
        "traffic_by_kernel": traffic.get("c2_fwd_bytes_by_kernel"),
        "algorithmic_bytes_per_launch": fwd_bytes,
        "share_of_step": r["fwd_ms"] / ms_step,
        # the forward is issue-bound: pipe utilisation from the ncu capture
        "pipes_ncu": traffic.get("c2_fwd_pipes"),
        "issue": issue_roofline(traffic.get("c2_fwd_warp_instr_per_launch"), r["fwd_ms"], peaks),
        "other_kernel": {"name": "bwd (k_row_bwd_w<float,16,2>)", "achieved": bwd_gbs, "frac": bwd_gbs / peak,
                         "traffic": traffic.get("c2_bwd_bytes_per_launch")},
    }
    e_ms, h2d, d2h = bench_c2_e2e(args, r["host"], ws, local)
    e2e = {"value": rows_total / (e_ms * 1e-3), "unit": "rows/s", "h2d_bytes_per_step": h2d * ws,
           "d2h_bytes_per_step": d2h * ws, "ms_per_step": e_ms, "ranks": ws,
           "pipeline": "per rank: 8 row blocks over 2 CUDA streams (H2D / kernels / D2H overlap)"}
    configs = None if args.no_configs else bench_configs(args, ws, rank, local, peak)
    ver = verify(r, ws, rank, local, with_c5=not args.no_configs) if args.verify else None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
    if rank == 0:
        passes = load_profile_json("ncu_passes_c5.json")
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, SURVEY 8(d) recipe)",
            "config": {"workload": WORKLOAD, "rows_per_gpu": C2_ROWS, "n": C2_N, "lam": "per-row softplus(U(-2,1))",
                       "global_batch": rows_total,
                       "parallelism": "dp%d (rank r owns rows [r*65536, (r+1)*65536); no collective)" % ws,
                       "l2": "no flush: every tensor (256 MiB) > L2 (126 MB)"},
            "fwd_ms": r["fwd_ms"], "bwd_ms": r["bwd_ms"],
            "fwd_ms_median": r["fwd_ms_median"], "bwd_ms_median": r["bwd_ms_median"],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": r["launches"],
            "clocks": r["clocks"], "pn_iterations": r["iters"], "configs": configs,
            "r2_per_pass_c5": passes or None, "verify": ver,
        }
        if configs:
            c5 = configs["C5"]
            line["secondary"] = {"metric": "2D TV prox fwd+bwd Mpixel/s (C5: 256x3x224x224, per-channel lambda, K=4)",
                                 "value": c5["value"], "unit": "Mpixel/s",
                                 "ms_per_step": c5["fwd_ms"]["mean"] + c5["bwd_ms"]["mean"]}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The CPU oracle timed as the reference arm (there is no reference implementation to
    install: /root/reference holds only the paper).  Rank 0 only under torchrun."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2204_03643_b200 import workloads
    oracle.build()
    cores = os.cpu_count() or 1
    rows = 16384                  # per step: large enough that the per-call thread team amortises
    w = workloads.c2(batch=rows * 2)

    def step(b):
        sl = slice((b % 2) * rows, (b % 2 + 1) * rows)
        x, brk, sgn = oracle.prox1d_batch(w.y[sl].astype(np.float64), w.lam[sl], nthreads=cores)
        oracle.bwd1d_batch(brk, sgn, w.grad[sl].astype(np.float64), nthreads=cores)

    for b in range(args.warmup):
        step(b)
    t0 = time.perf_counter()
    for b in range(args.steps):
        step(b)
    el = time.perf_counter() - t0
    value = rows * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY 8(d) recipe)",
        "config": {"workload": WORKLOAD, "rows_per_step": rows,
                   "note": "the CPU oracle (fp64 C taut string + segment mean) stands in for the reference: "
                           "there is no reference implementation (DESIGN.md)"},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "oracle",
                         "sample": "%d C2 rows per step, %d steps, %d threads" % (rows, args.steps, cores),
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="C2 headline only (profiling runs)")
    ap.add_argument("--verify", dest="verify", action="store_true", default=True,
                    help="gather outputs to rank 0 and compare (default on)")
    ap.add_argument("--no-verify", dest="verify", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if ws_env is not None and int(ws_env) != args.gpus:
        sys.exit("bench.py: WORLD_SIZE=%s but --gpus %d" % (ws_env, args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
