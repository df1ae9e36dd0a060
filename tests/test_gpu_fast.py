"""GPU parity of the fused window-pass path (uniform rank 16, leaves multiple of 16)
against the CPU oracle: every pass layout (L = 1..9, odd / even L, all lc), op N / C / T,
permuted rows and columns, ragged nrhs, and config 5 full-vector agreement with the
generic batched path."""
import numpy as np
import pytest
import torch

import oracle
from bfinputs import random_butterfly, random_rhs
import paper_2007_00202_b200 as pkg

pytestmark = pytest.mark.gpu


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X).T)).cuda()


def host(Y):
    torch.cuda.synchronize()
    return Y.cpu().numpy().T


TOL = {np.complex128: 1e-12, np.complex64: 1e-5}


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,leaf,lc", [(1, 16, None), (2, 16, None), (3, 32, None), (4, 16, None), (5, 16, None),
                                       (6, 16, None), (7, 16, None), (8, 16, None), (9, 16, None), (6, 16, 1),
                                       (6, 16, 5), (5, 64, 0), (5, 16, 5), (4, 32, 3)])
def test_fast_layouts(L, leaf, lc, dtype):
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=L * 10 + leaf, lc=lc, dtype=dtype)
    rng = np.random.default_rng(L)
    bf.row_perm = rng.permutation(bf.m).astype(np.int64)
    bf.col_perm = rng.permutation(bf.n).astype(np.int64)
    h = pkg.BFHandle(bf)
    assert h.rounds("N")[0]["name"].startswith("k_bf_pass"), h.rounds("N")
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 32), ("C", 45), ("T", 7)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=L + nr, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,nrhs,leaf", [(6, 1000, 16), (7, 700, 16), (5, 64 * 32 + 5, 16), (6, 1000, 64), (7, 640, 32)])
def test_fast_many_items(L, nrhs, leaf, dtype):
    """More work items (windows x rhs tiles) than SMs: each persistent CTA loops over
    several items, exercising the window / factor-ring buffer recycling."""
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=L, dtype=dtype)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    for op in "NC":
        X = random_rhs(bf.n, nrhs, seed=L + 1, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_fast_vs_generic_cfg5(monkeypatch, dtype):
    from bfinputs.configs import cfg5
    bf, X = cfg5(dtype)
    hf = pkg.BFHandle(bf)
    Xd = dev(X)
    Yf = hf.apply(Xd)
    Yfa = hf.apply(Xd, "C")
    del hf
    monkeypatch.setenv("BF_DISABLE_FAST", "1")
    hg = pkg.BFHandle(bf)
    assert hg.rounds("N")[0]["name"].startswith("k_stage_generic")
    Yg = hg.apply(Xd)
    Yga = hg.apply(Xd, "C")
    torch.cuda.synchronize()
    tol = 1e-13 if dtype == np.complex128 else 1e-5
    assert (torch.linalg.norm(Yf - Yg) / torch.linalg.norm(Yg)).item() <= tol
    assert (torch.linalg.norm(Yfa - Yga) / torch.linalg.norm(Yga)).item() <= tol
