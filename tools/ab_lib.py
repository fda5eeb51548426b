import sys, os, importlib
sys.path.insert(0, '.')
from paper_2204_03643_b200 import _lib
_lib.load(sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
import runpy
runpy.run_path('tools/time_kernels.py', run_name='__main__')
