#!/usr/bin/env python
"""Benchmark of the batched TV-prox hot path on B200 (arXiv 2204.03643).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one rank per GPU, NCCL)

Headline (`value`): BASELINE.json configs[1] = C2, batched 1D TV prox fwd+bwd,
65536 rows x 1024 samples, per-row lambda, fp32 -> rows/s over all ranks.  A
step = one forward (projected-Newton prox + saved mask) and one backward
(segment-mean VJP + per-row lambda gradient) over the whole batch; inputs
resident in HBM; every tensor (256 MiB) exceeds L2 (126 MB), so no flush is
needed.  Weak scaling: every rank runs its own full C2 batch; no collective on
the data path (rows are independent problems), NCCL only for the barrier and
the max-over-ranks timing reduction.
`secondary`: C5 (2D TV prox, 256x3x224x224, per-channel lambda, K=4) fwd+bwd
Mpixel/s, images sharded over ranks (strong scaling).
`e2e`: the same C2 metric through the public API with pinned host buffers,
H2D of y/lambda/grad_x and D2H of x/grad_y/grad_lambda inside the timed region.
`cpu_baseline`: the CPU oracle (oracle/, fp64 C) on a bounded sample of C2 rows
on the host cores (rank 0, N = 1 only).
`--impl reference`: the oracle timed as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
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
WORKLOAD = "C2: batched 1D TV prox fwd+bwd, 65536 x 1024, per-row lambda, fp32 (BASELINE.json configs[1])"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


def load_traffic():
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
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


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        if torch.cuda.is_available():
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
    torch.cuda.synchronize()


# --------------------------------------------------------------------------- ours
def bench_c2(args, ws, rank, local):
    import torch
    from paper_2204_03643_b200 import _lib, tvprox, workloads
    lib = _lib.load()
    w = workloads.c2()
    dev = torch.device("cuda", local)
    y = torch.as_tensor(w.y, device=dev)
    lam = torch.as_tensor(w.lam.astype(np.float32), device=dev)
    g = torch.as_tensor(w.grad, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        x, mask, _ = tvprox.tv1d_fwd(y, lam, need_mask=True)
        if ev is not None:
            ev[1].record(stream)
        gy, gl = tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW, want_lam=True)
        if ev is not None:
            ev[2].record(stream)
        return x, gy, gl

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clk = ClockSampler(local)
    clk.start()
    time.sleep(1.0)          # let nvidia-smi finish its NVML start-up before the timed region
    # warm-up right before the timed region (no idle gap: clocks ramp down when idle)
    # (outputs held across steps exactly as in the timed loop, so the caching allocator
    # owns every block it needs before timing starts: no cudaMalloc inside the region)
    out = None
    for _ in range(args.warmup):
        out = step()
    lib.tvp_launch_count(1)
    barrier(ws)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
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
    print("[bench] per-step fwd ms: %s" % " ".join("%.3f" % v for v in fwd_ms), file=sys.stderr)
    print("[bench] per-step bwd ms: %s" % " ".join("%.3f" % v for v in bwd_ms), file=sys.stderr)
    ms_max = allreduce_max(ms, ws)
    # iteration statistics (outside the timed region)
    _, _, it = tvprox.tv1d_fwd(y, lam, need_mask=False, want_iters=True)
    itn = it.cpu().numpy()
    del out
    return {
        "ms": ms_max, "ms_local": ms, "fwd_ms": statistics.mean(fwd_ms), "bwd_ms": statistics.mean(bwd_ms),
        "fwd_ms_median": statistics.median(fwd_ms), "bwd_ms_median": statistics.median(bwd_ms),
        "launches": launches, "clocks": clocks,
        "iters": {"mean": float(np.mean(itn & 0xFFFF)), "p99": float(np.percentile(itn & 0xFFFF, 99)),
                  "max": int((itn & 0xFFFF).max()), "not_converged": int((itn < 0).sum()),
                  "stall_accepts": int(((itn > 0) & ((itn >> 16) & 1 == 1)).sum())},
        "host": (w.y, w.lam.astype(np.float32), w.grad),
    }


def bench_c2_e2e(args, host, local, chunks=8):
    """Public-API end-to-end: pinned host -> device, fwd+bwd, device -> pinned host, every step.

    The batch is streamed in `chunks` row blocks over two CUDA streams, so the H2D copy
    of block i+1, the kernels of block i and the D2H copy of block i-1 overlap (rows are
    independent problems; PCIe is full duplex).  Every byte of every step's inputs and
    results still crosses the bus inside the timed region.
    """
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
    torch.cuda.synchronize()
    k = max(2, min(args.steps, 8))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for _ in range(k):
        step()
    t1.record(main)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / k
    h2d = y_h.numel() * 4 + l_h.numel() * 4 + g_h.numel() * 4
    d2h = x_o.numel() * 4 + gy_o.numel() * 4 + gl_o.numel() * 4
    return ms, h2d, d2h


def bench_c5(args, ws, rank, local):
    import torch
    from paper_2204_03643_b200 import _lib, tvprox, workloads
    off, per = shard(256, ws, rank)
    w = workloads.c5(N=per, image_offset=off)
    dev = torch.device("cuda", local)
    X = torch.as_tensor(w.X, device=dev)
    lam = torch.as_tensor(w.lam.astype(np.float32), device=dev)
    G = torch.as_tensor(w.grad, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        Y, saved, _ = tvprox.tv2d_fwd(X, lam, 4, training=True)
        if ev is not None:
            ev[1].record(stream)
        GX, gl = tvprox.tv2d_bwd(G, saved, _lib.LAM_PER_CHANNEL, 4, want_lam=True)
        if ev is not None:
            ev[2].record(stream)
        return Y, GX

    out = None
    for _ in range(max(2, args.warmup)):
        out = step()
    barrier(ws)
    k = max(3, min(args.steps, 10))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(k)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier(ws)
    t0.record(stream)
    for i in range(k):
        out = step(evs[i])
    t1.record(stream)
    barrier(ws)
    ms = allreduce_max(t0.elapsed_time(t1) / k, ws)
    _, _, it = tvprox.tv2d_fwd(X, lam, 4, training=False, want_iters=True)
    px_total = 256 * 3 * 224 * 224
    return {
        "metric": "2D TV prox fwd+bwd Mpixel/s (C5: 256x3x224x224, per-channel lambda, K=4, fp32)",
        "value": px_total / (ms * 1e-3) / 1e6, "unit": "Mpixel/s", "ms_per_step": ms,
        # one pixel = one NCHW element; the spatial rate counts N*H*W (3 channels per pixel)
        "spatial_mpx_per_s": px_total / 3 / (ms * 1e-3) / 1e6,
        "fwd_ms": statistics.mean(e[0].elapsed_time(e[1]) for e in evs),
        "bwd_ms": statistics.mean(e[1].elapsed_time(e[2]) for e in evs),
        "scaling": "strong", "images_per_rank": per,
        "max_pn_iters_per_pass": it.cpu().numpy().tolist(),
    }


def cpu_baseline(seconds=12.0, rows_per_batch=2048):
    """The oracle as it stands on the host cores: C2 rows fwd (taut string) + bwd (segment mean)."""
    import oracle
    from paper_2204_03643_b200 import workloads
    cores = os.cpu_count() or 1
    w = workloads.c2(batch=rows_per_batch * 4, with_grad=True)
    oracle.build()
    done, t_start = 0, time.perf_counter()
    b = 0
    while True:
        sl = slice((b % 4) * rows_per_batch, (b % 4 + 1) * rows_per_batch)
        y = w.y[sl].astype(np.float64)
        x, brk, sgn = oracle.prox1d_batch(y, w.lam[sl], nthreads=cores)
        oracle.bwd1d_batch(brk, sgn, w.grad[sl].astype(np.float64), nthreads=cores)
        done += rows_per_batch
        b += 1
        el = time.perf_counter() - t_start
        if el >= seconds:
            break
    return {"value": done / el, "unit": "rows/s", "cores": cores, "kind": "oracle",
            "sample": "%d C2 rows (1024 samples, per-row lambda) fwd+bwd in %.1f s, fp64 C oracle, %d threads"
                      % (done, el, cores)}


def issue_roofline(warp_instr, ms, peaks):
    """Instruction-issue roofline of the forward op: the executed warp instructions of one
    launch (ncu, committed profile) over its live duration, against the SM issue peak
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
    ws, rank, local = dist_setup(args)
    peak, peak_src, peaks = load_peaks()
    traffic = load_traffic()
    r = bench_c2(args, ws, rank, local)
    rows_total = C2_ROWS * ws
    value = rows_total / (r["ms"] * 1e-3 / args.steps)
    ms_step = r["ms"] / args.steps
    # roofline of the dominant kernel (the forward PN kernel): algorithmic bytes per launch
    per_row = 2 * C2_N * 4 + 4 + 4 * 64          # read y, read lambda, write x, write 2-bit mask
    fwd_bytes = C2_ROWS * per_row
    bwd_bytes = C2_ROWS * (2 * C2_N * 4 + 4 * 64 + 4)   # read grad_x + mask, write grad_y, grad_lambda
    fwd_gbs = fwd_bytes / (r["fwd_ms"] * 1e-3) / 1e9
    bwd_gbs = bwd_bytes / (r["bwd_ms"] * 1e-3) / 1e9
    dom = "fwd" if r["fwd_ms"] >= r["bwd_ms"] else "bwd"
    roof = {
        "kernel": "tv1d_prox_fwd = k_coarse_rows (coarse bound set) + k_row_fwd_w<float,16,2> (projected "
                  "Newton, 2 warps/line)" if dom == "fwd" else "k_row_bwd_w (1D segment-mean backward)",
        "bound": "hbm", "achieved": fwd_gbs if dom == "fwd" else bwd_gbs, "peak": peak, "unit": "GB/s",
        "frac": (fwd_gbs if dom == "fwd" else bwd_gbs) / peak, "peak_source": peak_src,
        "traffic": traffic.get("c2_fwd_bytes_per_launch" if dom == "fwd" else "c2_bwd_bytes_per_launch"),
        "algorithmic_bytes_per_launch": fwd_bytes if dom == "fwd" else bwd_bytes,
        "share_of_step": (r["fwd_ms"] if dom == "fwd" else r["bwd_ms"]) / ms_step,
        # the forward is issue-bound: pipe utilisation from the ncu capture
        "pipes_ncu": traffic.get("c2_fwd_pipes" if dom == "fwd" else "c2_bwd_pipes"),
        "issue": issue_roofline(traffic.get("c2_fwd_warp_instr_per_launch"), r["fwd_ms"], peaks) if dom == "fwd"
        else None,
        "other_kernel": {"name": "bwd" if dom == "fwd" else "fwd",
                         "achieved": bwd_gbs if dom == "fwd" else fwd_gbs,
                         "frac": (bwd_gbs if dom == "fwd" else fwd_gbs) / peak,
                         "traffic": traffic.get("c2_bwd_bytes_per_launch" if dom == "fwd" else "c2_fwd_bytes_per_launch")},
    }
    sec = bench_c5(args, ws, rank, local)
    c5_px = 256 * 3 * 224 * 224
    sec["roofline_whole_op"] = {"algorithmic_bytes": 2 * c5_px * 10 // ws,
                                "frac": (2 * c5_px * 10 / ws) / (sec["ms_per_step"] * 1e-3) / 1e9 / peak}
    e2e = None
    if rank == 0:
        e_ms, h2d, d2h = bench_c2_e2e(args, r["host"], local)
        e2e = {"value": C2_ROWS / (e_ms * 1e-3), "unit": "rows/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms, "ranks": 1,
               "pipeline": "8 row blocks over 2 CUDA streams (H2D / kernels / D2H overlap)"}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, SURVEY 8(d) recipe)",
            "config": {"workload": WORKLOAD, "rows_per_gpu": C2_ROWS, "n": C2_N, "lam": "per-row softplus(U(-2,1))",
                       "global_batch": rows_total, "parallelism": "dp%d (rows sharded, no collective)" % ws,
                       "l2": "no flush: every tensor (256 MiB) > L2 (126 MB)"},
            "fwd_ms": r["fwd_ms"], "bwd_ms": r["bwd_ms"],
            "fwd_ms_median": r["fwd_ms_median"], "bwd_ms_median": r["bwd_ms_median"],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": r["launches"],
            "clocks": r["clocks"], "pn_iterations": r["iters"], "secondary": sec,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2204_03643_b200 import workloads
    oracle.build()
    cores = os.cpu_count() or 1
    rows = 1024
    w = workloads.c2(batch=rows * 4)

    def step(b):
        sl = slice((b % 4) * rows, (b % 4 + 1) * rows)
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
                         "sample": "%d C2 rows per step, %d steps" % (rows, args.steps)},
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
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
