import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle
from paper_2204_03643_b200 import tvprox, workloads
from tests._util import unpack_codes, codes_to_brk_sgn
np.set_printoptions(linewidth=200, precision=3, suppress=True)
for dt in (torch.float32, torch.float64):
    n = 33; b = 4
    y = workloads.random_rows(9000 + n, b, n, "step", np.float64)
    lam = np.full(b, 0.5)
    yt = torch.as_tensor(y, dtype=dt, device='cuda')
    x, mask, it = tvprox.tv1d_fwd(yt, torch.as_tensor(lam, dtype=dt, device='cuda'), want_iters=True)
    g = np.random.default_rng(1).standard_normal((b, n))
    gy, gl = tvprox.tv1d_bwd(torch.as_tensor(g, dtype=dt, device='cuda'), mask, 1)
    torch.cuda.synchronize()
    codes = unpack_codes(mask.cpu().numpy(), n)
    brk, sgn = codes_to_brk_sgn(codes)
    gyr, glr = oracle.bwd1d_batch(brk, sgn, g)
    print(dt, "codes row0", codes[0])
    print("gy  ", gy.cpu().numpy()[0])
    print("ref ", gyr[0])
    print("g   ", g[0])
    print("err", np.abs(gy.cpu().numpy() - gyr).max(), "gl", gl.cpu().numpy(), glr)
