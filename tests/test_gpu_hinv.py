"""GPU parity of the HOD-BF inversion (hodbf_invert: Alg. 4 HODBF_invert with BF_SMW, P:569-615;
SURVEY 8(f) NEXT-3) against dense inverses from the CPU oracle's assembly (oracle.hodbf_dense).

Pins: zero off-diagonals -> blkdiag(D_t^{-1}) (Alg. 4 degenerates to line 3); a 2 x 2 block
matrix with dense (L = 0) off-diagonal blocks -> the exact 2 x 2 block inverse; constructed
Helmholtz HOD-BF matrices -> A^{-1} X against numpy.linalg.solve within the compression
tolerance, through the full BF_SMW recursion (dense_max = 0) and with dense small nodes; the
adjoint; and the Schur product F21 F11^{-1} F12 of Alg. 5 recompressed by
bf_random_matvec through the inverse.
"""
import numpy as np
import pytest
import torch

import oracle
from bfinputs import Stage, butterfly_from_blocks, random_rhs
from bfinputs.factors import HODBF
from bfinputs.configs import helmholtz_plane_hodbf, helmholtz_planes_bf
import paper_2007_00202_b200 as pkg
from paper_2007_00202_b200 import construct as cx

pytestmark = pytest.mark.gpu


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X).T)).cuda()


def host(Y):
    torch.cuda.synchronize()
    return Y.cpu().numpy().T


def _L0(A):
    m, n = A.shape
    return butterfly_from_blocks(0, 0, [0, m], [0, n], np.arange(m), np.arange(n), [np.eye(m)], {}, [A], {},
                                 [np.eye(n)])


def test_zero_offdiag_is_blockdiag_inverse():
    rng = np.random.default_rng(0)
    LH, leaf = 3, 5
    n = leaf << LH
    lp = np.arange((1 << LH) + 1) * leaf
    Ds = [rng.standard_normal((leaf, leaf)) + 1j * rng.standard_normal((leaf, leaf)) + 4 * np.eye(leaf)
          for _ in range(1 << LH)]
    off = [[_L0(np.zeros((leaf << (LH - l), leaf << (LH - l)))) for _ in range(1 << l)] for l in range(1, LH + 1)]
    perm = rng.permutation(n)
    H = HODBF(n, LH, lp, perm, Stage.from_blocks(Ds, np.complex128), off)
    inv = cx.HODBFInverse(H, eps=1e-12)
    assert inv.nbutterflies == 0
    A = oracle.hodbf_dense(H)
    X = random_rhs(n, 4, seed=1)
    for op, M in (("N", A), ("C", A.conj().T)):
        assert oracle.rel_err(host(inv.apply(dev(X), op)), np.linalg.solve(M, X)) <= 1e-13


def test_two_by_two_dense_blocks():
    """L_H = 1, off-diagonal blocks dense (L = 0 butterflies): the inverse is the exact 2 x 2 block
    inverse (BF_SMW at L = 0 is the dense SMW)."""
    rng = np.random.default_rng(1)
    n1, n2 = 7, 9
    A = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16)) + 6 * np.eye(16)
    lp = np.array([0, n1, 16])
    H = HODBF(16, 1, lp, np.arange(16), Stage.from_blocks([A[:n1, :n1], A[n1:, n1:]], np.complex128),
              [[_L0(A[:n1, n1:]), _L0(A[n1:, :n1])]])
    inv = cx.HODBFInverse(H, eps=1e-14, rank_max=16)
    X = random_rhs(16, 3, seed=2)
    assert oracle.rel_err(host(inv.apply(dev(X))), np.linalg.solve(A, X)) <= 1e-12
    assert oracle.rel_err(host(inv.apply(dev(X), "C")), np.linalg.solve(A.conj().T, X)) <= 1e-12


@pytest.mark.parametrize("dense_max", [0, 64])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_helmholtz_hodbf_inverse(dense_max, dtype):
    """A constructed Helmholtz HOD-BF (16 x 16 grid, leaf 16, L_H = 4, eps 1e-4 compression):
    A^{-1} X and A^{-H} X against numpy.linalg.solve on the assembled matrix, and the residual
    ||A (A^{-1} X) - X|| (the HOD-BF apply is the library's)."""
    H = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4).astype(dtype)
    eps = 1e-10 if dtype == np.complex128 else 1e-5
    inv = cx.HODBFInverse(H, eps=eps, rank_max=64, dense_max=dense_max)
    assert inv.stats["saturated"] == 0, inv.stats
    A = oracle.hodbf_dense(H)
    X = random_rhs(H.n, 8, seed=3, dtype=dtype)
    tol = 1e-7 if dtype == np.complex128 else 1e-3
    for op, M in (("N", A), ("C", A.conj().T)):
        ref = np.linalg.solve(M, X.astype(np.complex128))
        assert oracle.rel_err(host(inv.apply(dev(X), op)), ref) <= tol, op
    h = pkg.HODBFHandle(H)
    Y = inv.apply(dev(X))
    R = h.apply(Y)
    assert oracle.rel_err(host(R), X) <= tol


def test_schur_product_through_inverse():
    """Alg. 5 line S_construction: S = F21 F11^{-1} F12 with F11 an HOD-BF (the plane's
    self-interaction), F12 = K^H and F21 = K for the Helmholtz butterfly K between the plane and a
    parallel one; recompressed by bf_random_matvec on K's row trees, against the dense product."""
    F11 = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4)
    K = helmholtz_planes_bf(16, 16, 10.0, 8.0, 1e-8)
    inv = cx.HODBFInverse(F11, eps=1e-10, rank_max=64)
    hK = pkg.BFHandle(K)
    op = cx.Operator(K.m, K.m, np.complex128, [(1.0, [(hK, "C"), (inv, "N"), (hK, "N")], 0, 0)])
    eps = 1e-7
    res = cx.random_matvec(op, K.m, K.m, K.L, K.row_leaf_ptr, K.row_leaf_ptr, K.row_perm, K.row_perm,
                           eps=eps, rank_max=100, oversample=12, seed=5)
    Kd = oracle.bf_dense(K)
    S = Kd @ np.linalg.solve(oracle.hodbf_dense(F11), Kd.conj().T)
    Srec = oracle.bf_dense(cx.export(res.handle, res.trees))
    err = np.linalg.norm(Srec - S) / np.linalg.norm(S)
    assert err <= 10 * eps + 1e-8, (err, res.stats)
