"""Run bench.bench_c2 repeatedly (the bench's own step) and report per-step outliers,
with the nvidia-smi sampler on (default) or off (BENCH_NO_SAMPLER=1)."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
if os.environ.get("BENCH_NO_SAMPLER"):
    class _Null:
        def __init__(self, i): pass
        def start(self): pass
        def stop(self): return {}
    bench.ClockSampler = _Null
args = argparse.Namespace(steps=int(os.environ.get("STEPS", "20")), warmup=5)
ws, rank, local = bench.dist_setup(args)
for rep in range(6):
    r = bench.bench_c2(args, ws, rank, local)
    print("rep %d ms/step %.4f fwd mean %.4f median %.4f" % (rep, r["ms"] / args.steps, r["fwd_ms"], r["fwd_ms_median"]), flush=True)
