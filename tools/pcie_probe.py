"""Pinned H2D / D2H bandwidth and the bench e2e step with different chunk / stream counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import numpy as np
import torch
import bench
from paper_2204_03643_b200 import workloads

n = 256 << 20
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): fn()
    b.record(); torch.cuda.synchronize()
    print("%s %.1f GB/s" % (name, 5 * n / (a.elapsed_time(b) * 1e-3) / 1e9))
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
h2 = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("both directions concurrently: %.1f GB/s each" % (5 * n / (time.perf_counter() - t0) / 1e9))
w = workloads.c2()
host = (w.y, w.lam.astype(np.float32), w.grad)
args = argparse.Namespace(steps=8, warmup=3)
for chunks in (4, 8, 16, 32):
    ms, h2d, d2h = bench.bench_c2_e2e(args, host, 0, chunks=chunks)
    print("chunks %2d: %.2f ms/step -> %.2f M rows/s" % (chunks, ms, 65536 / ms / 1e3))
