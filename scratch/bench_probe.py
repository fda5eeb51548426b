"""Per-step fwd/bwd event times of the C2 bench loop under different conditions
(nvidia-smi sampler on/off, idle gap before timing) -- diagnosing bench inflation."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import _lib, tvprox, workloads  # noqa: E402

w = workloads.c2()
y = torch.as_tensor(w.y, device="cuda")
lam = torch.as_tensor(w.lam.astype(np.float32), device="cuda")
g = torch.as_tensor(w.grad, device="cuda")
s = torch.cuda.current_stream()


def run(tag, sampler, gap, steps=20):
    p = None
    if sampler:
        p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.DEVNULL)
    time.sleep(gap)
    for _ in range(5):
        x, mask, _ = tvprox.tv1d_fwd(y, lam)
        tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    h0 = time.perf_counter()
    for i in range(steps):
        ev[i][0].record(s)
        x, mask, _ = tvprox.tv1d_fwd(y, lam)
        ev[i][1].record(s)
        tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW)
        ev[i][2].record(s)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    if p:
        p.terminate()
    f = [e[0].elapsed_time(e[1]) for e in ev]
    b = [e[1].elapsed_time(e[2]) for e in ev]
    f = np.array(f); b = np.array(b)
    med = np.median(f)
    print("%-22s steps %d wall %.1f ms | fwd median %.3f max %.3f outliers(>1.2x) %d | bwd max %.3f" % (
        tag, steps, (h2 - h0) * 1e3, med, f.max(), int((f > 1.2 * med).sum()), b.max()), flush=True)


for rep in range(2):
    run("no-sampler", False, 0.5, steps=300)
    run("sampler-100ms", True, 1.0, steps=300)
