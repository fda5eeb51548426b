"""Build libtvprox.so (sm_100a) in-tree with nvcc.

    python -m paper_2204_03643_b200.build [--force] [--verbose]

Compiles each translation unit of csrc/ in parallel with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and links them with a
static cudart into ``paper_2204_03643_b200/libtvprox.so``.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libtvprox.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu*")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, debug: bool = False,
          defines=(), out: str = None) -> str:
    """debug=True builds libtvprox_debug.so with -DTVP_DEBUG (per-iteration device printf).
    defines/out: a tuning variant (-D flags) built into its own directory and library (A/B only)."""
    bdir = BUILD + ("_debug" if debug else "")
    lib = LIB.replace(".so", "_debug.so") if debug else LIB
    if out:
        bdir = BUILD + "_" + os.path.splitext(os.path.basename(out))[0]
        lib = os.path.abspath(out)
    os.makedirs(bdir, exist_ok=True)
    deps = _deps()
    if not force and not _stale(lib, deps):
        return lib
    objs = []
    jobs = []
    for src in _sources():
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, deps):
            cmd = [NVCC] + ARCH + FLAGS + (["-Xptxas", "-v"] if ptxas_v else []) + \
                (["-DTVP_DEBUG"] if debug else []) + ["-D" + d for d in defines] + ["-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        p = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, p

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for cmd, p in ex.map(run, jobs):
            if verbose or p.returncode:
                sys.stderr.write(p.stdout + p.stderr)
            if p.returncode:
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = lib + ".tmp%d" % os.getpid()
    link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true")
    ap.add_argument("--debug", action="store_true")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, ptxas_v=a.ptxas, debug=a.debug, defines=a.define, out=a.out))
