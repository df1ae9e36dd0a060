"""Pins of the multifrontal sweep oracle (oracle/mf.py).  No GPU.

  * with F12 = F21 = 0 the sweep is the block-diagonal solve of the separator blocks F11;
  * on a synthetic assembly tree, the forward / backward substitution equals the dense solve of
    the assembled block-LU matrix M = L U (lower: F11 on (s, s), F21 on (u, s); upper: I plus
    F11^{-1} F12 on (s, u)), and the tree's index structure is the multifrontal one (post-order,
    update sets inside the parent's front).
"""
import numpy as np

from bfinputs import random_rhs
from bfinputs.fronts import synthetic_fronts
from oracle.mf import mf_matrix, mf_solve
from oracle.dense import hodbf_dense


def test_fronts_structure():
    fronts, N = synthetic_fronts(depth=2, nx_leaf=4, seed=1)
    assert sum(f.s_len for f in fronts) == N and fronts[-1].parent == -1
    for k, f in enumerate(fronts):
        if f.parent >= 0:
            p = fronts[f.parent]
            assert f.parent > k
            pool = set(range(p.s_off, p.s_off + p.s_len)) | set(p.u_idx.tolist())
            assert set(f.u_idx.tolist()) <= pool


def test_sweep_without_coupling_is_blockdiag_solve():
    fronts, N = synthetic_fronts(depth=2, nx_leaf=4, seed=2, coupling=0.0)
    B = random_rhs(N, 3, seed=1)
    X = mf_solve(fronts, N, B)
    for f in fronts:
        s = slice(f.s_off, f.s_off + f.s_len)
        np.testing.assert_allclose(hodbf_dense(f.F11) @ X[s], B[s], rtol=0, atol=1e-12 * np.abs(B).max())


def test_sweep_equals_dense_block_lu_solve():
    fronts, N = synthetic_fronts(depth=2, nx_leaf=4, seed=3)
    B = random_rhs(N, 4, seed=2)
    M = mf_matrix(fronts, N)
    X = mf_solve(fronts, N, B)
    assert np.linalg.norm(M @ X - B) / np.linalg.norm(B) < 1e-12
