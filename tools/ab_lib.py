"""Run a timing script against a variant library (same-box A/B).

    python tools/ab_lib.py <lib.so> [tools/<script>.py] <script args...>
(default script: tools/time_kernels.py)
"""
import os
import runpy
import sys

sys.path.insert(0, '.')
from paper_2204_03643_b200 import _lib  # noqa: E402

_lib.load(sys.argv[1])
script = 'tools/time_kernels.py'
rest = sys.argv[2:]
if rest and rest[0].endswith('.py'):
    script, rest = rest[0], rest[1:]
sys.argv = [script] + rest
runpy.run_path(script, run_name='__main__')
