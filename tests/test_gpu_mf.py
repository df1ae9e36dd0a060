"""GPU parity of the multifrontal solve-phase sweep (bf_mf_solve)
against the CPU oracle's sweep (oracle/mf.py) on seeded synthetic assembly trees.

With every front's F11 inverted densely (dense_max >= the separator size) the GPU sweep and the
oracle compute the same map up to rounding: <= 1e-12 (complex128).  With F11^{-1} compressed by
hodbf_invert (eps 1e-10) the difference is the inversion tolerance.  nrhs = 1 (the solve regime)
and blocks of right-hand sides.
"""
import numpy as np
import pytest
import torch

from bfinputs import random_rhs
from bfinputs.fronts import synthetic_fronts
from oracle.mf import mf_solve
from oracle import rel_err
from paper_2007_00202_b200 import construct as cx

pytestmark = pytest.mark.gpu


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X).T)).cuda()


@pytest.mark.parametrize("nrhs", [1, 7, 32])
def test_mf_sweep_dense_fronts(nrhs):
    fronts, N = synthetic_fronts(depth=2, nx_leaf=8, seed=1)
    mf = cx.MFSolver(fronts, N, eps=1e-12, dense_max=4096)
    B = random_rhs(N, nrhs, seed=nrhs)
    X = mf.solve(dev(B)).cpu().numpy().T
    assert rel_err(X, mf_solve(fronts, N, B)) <= 1e-12


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_mf_sweep_compressed_inverses(dtype):
    fronts, N = synthetic_fronts(depth=2, nx_leaf=8, seed=2, dtype=dtype)
    mf = cx.MFSolver(fronts, N, eps=1e-10 if dtype == np.complex128 else 1e-5, rank_max=64)
    assert any(inv.nbutterflies > 0 for inv in mf.inv)
    B = random_rhs(N, 4, seed=3, dtype=dtype)
    X = mf.solve(dev(B)).cpu().numpy().T
    assert rel_err(X, mf_solve(fronts, N, B)) <= (1e-7 if dtype == np.complex128 else 1e-3)
