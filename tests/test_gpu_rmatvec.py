"""GPU parity of the randomized matrix-free construction (bf_random_matvec, SURVEY 8(f) NEXT-2;
PAPER.md Sec. 3.3) and of its building blocks.

The construction is not unique (pivot choices, sketches), so its result is judged against the
operator it compresses, densified by the CPU oracle (||A - B||_F <= c eps ||A||_F):
  * an exact rank-r random-factor butterfly (config-1 shape) is recovered to <= 1e-10;
  * a product F21 F12 of two config-2-shaped Helmholtz butterflies (P:685's Schur products are
    such operator products) is recompressed within 10 eps;
  * the zero operator gives the zero butterfly;
  * the batched ID kernel equals scipy's column-pivoted QR (ranks, pivots, R11^-1 R12).
"""
import numpy as np
import pytest
import scipy.linalg as sla
import torch

import oracle
from bfinputs import random_butterfly, random_rhs
from bfinputs.configs import helmholtz_planes_bf
import paper_2007_00202_b200 as pkg
from paper_2007_00202_b200 import construct as cx

pytestmark = pytest.mark.gpu


def rel(A, B):
    return np.linalg.norm(A - B) / np.linalg.norm(B)


def rebuild(res):
    return oracle.bf_dense(cx.export(res.handle, res.trees))


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,lc,perm", [(5, None, False), (5, None, True), (4, 0, True), (4, 4, False), (3, 1, True)])
def test_recover_random_butterfly(L, lc, perm, dtype):
    """A random-factor butterfly of exact rank 8 (config-1 shape: leaf 32, r = 8) applied through
    its own handle is recovered from sketches: ranks 8 everywhere and the dense matrices agree."""
    bf = random_butterfly(L=L, leaf=32, r=8, seed=L, lc=lc, dtype=dtype)
    if perm:
        bf.row_perm = np.random.default_rng(1).permutation(bf.m)
        bf.col_perm = np.random.default_rng(2).permutation(bf.n)
    h = pkg.BFHandle(bf)
    op = cx.Operator(bf.m, bf.n, dtype, [(1.0, [(h, "N")], 0, 0)])
    # complex64: the sketches carry ~1e-6 relative rounding through up to L stages of the apply, so
    # the truncation sits above that floor
    eps = 1e-12 if dtype == np.complex128 else 1e-5
    res = cx.random_matvec(op, bf.m, bf.n, bf.L, bf.row_leaf_ptr, bf.col_leaf_ptr, bf.row_perm, bf.col_perm,
                           lc=bf.lc, eps=eps, rank_max=12, oversample=8, seed=3, dtype=dtype)
    assert res.stats["saturated"] == 0, res.stats
    assert res.stats["max_rank"] == 8 if dtype == np.complex128 else res.stats["max_rank"] <= 10, res.stats
    err = rel(rebuild(res), oracle.bf_dense(bf))
    assert err <= (1e-10 if dtype == np.complex128 else 1e-4), err
    # the constructed butterfly applies like the original
    X = random_rhs(bf.n, 5, seed=4, dtype=dtype)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = res.handle.apply(Xd).cpu().numpy().T
    assert oracle.rel_err(Y, oracle.bf_apply(bf, X)) <= (1e-10 if dtype == np.complex128 else 1e-4)
    # matvec columns: (2^(lc+1) - 1) k adjoint, (2^(L-lc+1) - 1) k forward (P:450-452's O(sqrt(n)) sketches)
    k = 12 + 8
    lcv = bf.lc
    assert res.stats["matvec_cols_c"] == ((1 << (lcv + 1)) - 1) * k
    assert res.stats["matvec_cols_n"] == ((1 << (L - lcv + 1)) - 1) * k


def test_zero_operator():
    bf = random_butterfly(L=4, leaf=16, r=4, seed=0)
    h = pkg.BFHandle(bf)
    op = cx.Operator(bf.m, bf.n, np.complex128, [(0.0, [(h, "N")], 0, 0)])
    res = cx.random_matvec(op, bf.m, bf.n, bf.L, bf.row_leaf_ptr, bf.col_leaf_ptr, eps=1e-12, rank_max=8)
    assert res.stats["max_rank"] == 0
    assert np.abs(rebuild(res)).max() == 0


@pytest.mark.parametrize("eps", [1e-6, 1e-8])
def test_product_of_helmholtz_butterflies(eps):
    """F21 F12 with F12 = the config-2-shaped Helmholtz butterfly between two 32 x 32 planes (8h
    apart) and F21 = the adjoint of the same geometry at 6h: the product maps the z = 0 plane to
    itself; its recompression on the butterfly's column tree is within 10 eps of the dense
    product (both factors densified by the oracle)."""
    A1 = helmholtz_planes_bf(32, 64, 8.0, 8.0, 1e-6)
    A2 = helmholtz_planes_bf(32, 64, 8.0, 6.0, 1e-6)
    h1, h2 = pkg.BFHandle(A1), pkg.BFHandle(A2)
    D = oracle.bf_dense(A2).conj().T @ oracle.bf_dense(A1)
    op = cx.Operator(A2.n, A1.n, np.complex128, [(1.0, [(h1, "N"), (h2, "C")], 0, 0)])
    res = cx.random_matvec(op, A2.n, A1.n, A1.L, A2.col_leaf_ptr, A1.col_leaf_ptr, A2.col_perm, A1.col_perm,
                           eps=eps, rank_max=160, oversample=16, seed=7)
    assert res.stats["saturated"] == 0, res.stats
    err = rel(rebuild(res), D)
    assert err <= 10 * eps, (err, res.stats)


def test_operator_apply_sums_and_blocks():
    """bf_operator_apply: Y = (2 K1 - 1j K2^H K1) X placed blockwise, op N and C, against dense."""
    K1b = random_butterfly(L=3, leaf=8, r=3, seed=1)
    K2b = random_butterfly(L=3, leaf=8, r=3, seed=2)
    h1, h2 = pkg.BFHandle(K1b), pkg.BFHandle(K2b)
    n = K1b.n
    op = cx.Operator(2 * n, 2 * n, np.complex128,
                     [(2.0, [(h1, "N")], 0, 0), (-1j, [(h1, "N"), (h2, "C")], n, n), (0.5, [("I", n)], n, 0)])
    K1, K2 = oracle.bf_dense(K1b), oracle.bf_dense(K2b)
    A = np.zeros((2 * n, 2 * n), dtype=np.complex128)
    A[:n, :n] += 2 * K1
    A[n:, n:] += -1j * (K2.conj().T @ K1)
    A[n:, :n] += 0.5 * np.eye(n)
    X = random_rhs(2 * n, 6, seed=3)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    assert oracle.rel_err(op.apply(Xd, "N").cpu().numpy().T, A @ X) <= 1e-13
    assert oracle.rel_err(op.apply(Xd, "C").cpu().numpy().T, A.conj().T @ X) <= 1e-13


@pytest.mark.parametrize("dtype", [torch.complex128, torch.complex64])
def test_batched_id_vs_scipy(dtype):
    """bf_batched_id == scipy.linalg.qr(pivoting=True) truncated at |R_jj| <= eps |R_00|: ranks,
    pivots and T = R11^{-1} R12, on low-rank, full-rank, wide and tall complex matrices."""
    rng = np.random.default_rng(0)
    shapes = [(20, 30, 5), (20, 30, 20), (20, 12, 12), (40, 12, 12), (24, 64, 9), (24, 8, 3), (33, 70, 33)]
    mats, refs = [], []
    eps = 1e-10 if dtype == torch.complex128 else 1e-4
    for k, p, r in shapes:
        A = (rng.standard_normal((k, r)) + 1j * rng.standard_normal((k, r))) @ \
            (rng.standard_normal((r, p)) + 1j * rng.standard_normal((r, p)))
        mats.append(torch.from_numpy(np.ascontiguousarray(A.T)).to(dtype).cuda())
        A64 = np.asarray(A.astype(np.complex64 if dtype == torch.complex64 else np.complex128), dtype=np.complex128)
        Q, R, P = sla.qr(A64, pivoting=True, mode="economic")
        d = np.abs(np.diag(R))
        rr = int(np.sum(d > eps * d[0]))
        T = sla.solve_triangular(R[:rr, :rr], R[:rr, rr:])
        refs.append((rr, P, T))
    out = [None] * len(mats)
    for k in sorted({m.shape[1] for m in mats}):   # one sketch width per call
        sel = [i for i, m in enumerate(mats) if m.shape[1] == k]
        for i, o in zip(sel, cx.batched_id([mats[i] for i in sel], eps, 1000)):
            out[i] = o
    for (r, pm, T), (rr, P, Tr) in zip(out, refs):
        assert r == rr
        np.testing.assert_array_equal(pm[:r], P[:r])
        # T's columns belong to the redundant columns pm[r:] (resp. P[r:]); compare column by column
        assert sorted(pm[r:]) == sorted(P[r:])
        T = T[:, np.argsort(pm[r:])]
        Tr = Tr[:, np.argsort(P[r:])]
        tol = 1e-9 if dtype == torch.complex128 else 2e-2
        if T.size == 0:
            continue
        assert np.abs(T - Tr).max() <= tol * max(1.0, np.abs(Tr).max()), np.abs(T - Tr).max()
