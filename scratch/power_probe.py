"""Sustained-load probe: C2 forward back to back for ~3 s with nvidia-smi sampling
(clocks, power, throttle reasons) to see whether per-launch time drifts with clocks."""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import tvprox, workloads  # noqa: E402

w = workloads.c2()
y = torch.as_tensor(w.y, device="cuda")
lam = torch.as_tensor(w.lam.astype(np.float32), device="cuda")
lines = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu",
                      "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [lines.append((time.time(), l.strip())) for l in p.stdout], daemon=True)
th.start()
time.sleep(0.5)
for _ in range(3):
    tvprox.tv1d_fwd(y, lam)
torch.cuda.synchronize()
t_start = time.time()
evs = []
for i in range(900):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    tvprox.tv1d_fwd(y, lam)
    b.record()
    evs.append((a, b))
torch.cuda.synchronize()
t_end = time.time()
time.sleep(0.3)
p.terminate()
ts = np.array([a.elapsed_time(b) for a, b in evs])
for lo in range(0, len(ts), 100):
    print("launches %4d-%4d: mean %.3f ms min %.3f max %.3f" % (lo, lo + 99, ts[lo:lo + 100].mean(), ts[lo:lo + 100].min(), ts[lo:lo + 100].max()))
load = [l for t, l in lines if t_start <= t <= t_end]
print("samples under load:", len(load))
for l in load[:: max(1, len(load) // 15)]:
    print("  ", l)
