"""B200-native (sm_100a) batched TV proximity operators of arXiv 2204.03643.

The compute path is libtvprox.so (hand-written CUDA behind the C ABI in
include/tvprox.h).  Import the binding lazily:

    from paper_2204_03643_b200 import tvprox
    x = tvprox.tv1d(y, lam)            # autograd-aware
    Y = tvprox.tv2d(X, lam, iters=4)
"""
__all__ = ["tvprox", "workloads"]
