import numpy as np, sys, os
sys.path.insert(0,'.')
import oracle
from tests._util import codes_to_brk_sgn
print("cpus", os.cpu_count())
print(oracle._LIB, os.path.getmtime(oracle._LIB), os.path.getmtime(oracle._SRC))
rng=np.random.default_rng(0)
codes=rng.integers(0,3,(40,32)).astype(np.int8)
codes[:, :10]=0
brk,sgn=codes_to_brk_sgn(codes)
g=rng.standard_normal((40,33)).astype(np.float32)
outs=[oracle.bwd1d_batch(brk,sgn,g.astype(np.float64),nthreads=nt)[0] for nt in (1,8,1,8)]
print([np.abs(o-outs[0]).max() for o in outs])
gy0=np.array([oracle.bwd1d(brk[r],sgn[r],g[r].astype(np.float64))[0] for r in range(40)])
print(np.abs(gy0-outs[0]).max())
import torch
x=torch.zeros(3,device='cuda')
outs=[oracle.bwd1d_batch(brk,sgn,g.astype(np.float64),nthreads=nt)[0] for nt in (1,8,1,8)]
print("after torch cuda", [np.abs(o-gy0).max() for o in outs])
