"""Debug the complex64 tcgen05 tile kernel on small cases (prints per-op errors)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2007_00202_b200 as pkg  # noqa: E402
from bfinputs.factors import random_ranks_butterfly, random_rhs  # noqa: E402


def run(h, X, op):
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = h.apply(Xd, op)
    torch.cuda.synchronize()
    return Y.cpu().numpy().T


for (L, lc, rmin, rmax, nrhs) in [(1, 0, 16, 16, 64), (2, 1, 8, 8, 64), (3, 1, 1, 20, 64), (5, 2, 0, 70, 64)]:
    rng = np.random.default_rng(7)
    nb = 1 << L
    rows = rng.integers(16, 40, nb)
    cols = rng.integers(16, 40, nb)
    bf = random_ranks_butterfly(L, rows, cols, seed=7, rmin=rmin, rmax=rmax, lc=lc, dtype=np.complex64)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    for op in ("N", "C"):
        X = random_rhs(bf.n if op == "N" else bf.m, nrhs, seed=3, dtype=np.complex64)
        Y = run(h, X, op)
        R = oracle.apply_op(K, X, op)
        err = oracle.rel_err(Y, R)
        print(L, lc, rmin, rmax, op, "err", err, "Ynorm", np.linalg.norm(Y), "Rnorm", np.linalg.norm(R), flush=True)
        if err > 1e-5 and L <= 2:
            d = np.abs(Y - R)
            print("  max diff rows", np.argsort(-d.max(1))[:8], "cols", np.argsort(-d.max(0))[:8])
            print("  Y[0,:4]", Y[0, :4], "R[0,:4]", R[0, :4])
