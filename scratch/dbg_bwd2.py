import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle
from paper_2204_03643_b200 import tvprox, workloads
from tests._util import unpack_codes, codes_to_brk_sgn
np.set_printoptions(linewidth=220, precision=3, suppress=True)
n = 33
y = workloads.random_rows(9000 + n, 40, n, "step", np.float32)
lam = np.random.default_rng(n + 1).uniform(0.05, 1.0, 40).astype(np.float32)
yt = torch.as_tensor(y, device='cuda')
x, mask, it = tvprox.tv1d_fwd(yt, torch.as_tensor(lam, device='cuda'), want_iters=True)
g = np.random.default_rng(n).standard_normal((40, n)).astype(np.float32)
for variant in ("direct", "roundtrip"):
    m = mask if variant == "direct" else torch.as_tensor(mask.cpu().numpy(), device='cuda')
    gy, gl = tvprox.tv1d_bwd(torch.as_tensor(g, device='cuda'), m, 1)
    torch.cuda.synchronize()
    codes = unpack_codes(mask.cpu().numpy(), n)
    brk, sgn = codes_to_brk_sgn(codes)
    for nt in (1, 8):
        gyr, glr = oracle.bwd1d_batch(brk, sgn, g.astype(np.float64), nthreads=nt)
        e = np.abs(gy.cpu().numpy() - gyr)
        print(variant, nt, "err", e.max(), "worst row", e.max(1).argmax())
r = e.max(1).argmax()
print("codes", codes[r]); print("gy ", gy.cpu().numpy()[r]); print("ref", gyr[r]); print("g  ", g[r])
print("mask words", mask.cpu().numpy()[r], mask.shape, mask.dtype, mask.stride())
