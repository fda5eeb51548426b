import numpy as np, torch, sys, pickle
sys.path.insert(0, '.')
from paper_2204_03643_b200 import _lib
_lib.load(_lib.LIB_PATH.replace('.so', '_debug.so'))
from paper_2204_03643_b200 import tvprox
import oracle
d = pickle.load(open(sys.argv[1], 'rb'))[int(sys.argv[2])]
y = torch.as_tensor(d['y'][None, :].copy(), device='cuda')
warm = None if d['warm'] is None else torch.as_tensor(d['warm'][None, :].copy(), device='cuda')
x, m, it = tvprox.tv1d_fwd(y, d['lam'], want_iters=True, warm_mask=warm)
torch.cuda.synchronize()
ref = oracle.prox1d(d['y'].astype(np.float64), d['lam'])
print("status", hex(it.item()), "err", np.abs(x.cpu().numpy()[0] - ref).max())
