"""Pins of the CPU oracle against things fixed by the paper and by mathematics (no GPU).

Each test names the pin of DESIGN.md "Pins" it establishes:
  P1 identity closed form          P2 L = 0 reduces to the dense block
  P3 DFT closed form vs numpy.fft   P4 kernel compression within 10 eps of brute force
  P5 adjoint dot-product identity   P6 linearity / trivial inputs
  P7 blockwise Eq.(3.1)-(3.2) vs the product of explicit sparse factors Eq.(3.3)
  P8 HOD-BF structure               P9 sampled-row oracle == dense oracle rows
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from bfinputs import (Stage, butterfly_from_blocks, dft_butterfly, identity_butterfly,
                      random_butterfly, random_ranks_butterfly, random_rhs)
from bfinputs.factors import HODBF
from bfinputs.construct import col_id, row_id
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- P1
@pytest.mark.parametrize("L,m0", [(1, 1), (2, 1), (3, 1), (4, 2), (5, 4), (3, 3), (6, 2)])
def test_P1_identity_closed_form(L, m0):
    bf = identity_butterfly(L, m0)
    oracle.validate(bf)
    K = oracle.bf_dense(bf)
    np.testing.assert_array_equal(K, np.eye(bf.n))


def test_P1_identity_wrong_perm_is_not_identity():
    # the bit-reversed column tree is essential: with the natural order K != I
    bf = identity_butterfly(3, 1)
    bf.col_perm = np.arange(bf.n)
    assert not np.array_equal(oracle.bf_dense(bf), np.eye(bf.n))


# ---------------------------------------------------------------- P2
def test_P2_L0_is_dense_block():
    rng = np.random.default_rng(5)
    Bm = rng.standard_normal((7, 5)) + 1j * rng.standard_normal((7, 5))
    bf = butterfly_from_blocks(0, 0, [0, 7], [0, 5], np.arange(7), np.arange(5),
                               [np.eye(7)], {}, [Bm], {}, [np.eye(5)])
    oracle.validate(bf)
    np.testing.assert_array_equal(oracle.bf_dense(bf), Bm)


# ---------------------------------------------------------------- P3
def _dft_matrix(n):
    j = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(j, j) / n)


def test_P3_golden_dft4():
    # textbook 4-point DFT (F_jk = w^{jk}, w = e^{-2 pi i/4} = -i), tests/golden/dft4.txt
    F = np.loadtxt(os.path.join(GOLDEN, "dft4.txt"), dtype=str)
    F = np.array([[complex(v.replace("i", "j")) for v in row] for row in F])
    K = oracle.bf_dense(dft_butterfly(2))
    np.testing.assert_allclose(K, F, atol=1e-15)


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 6, 8, 10])
def test_P3_dft_closed_form(L):
    bf = dft_butterfly(L)
    oracle.validate(bf)
    n = 1 << L
    K = oracle.bf_dense(bf)
    F = np.fft.fft(np.eye(n), axis=0)
    assert np.abs(K - F).max() < 1e-13 * max(1, L)
    assert np.abs(K - _dft_matrix(n)).max() < 1e-12
    X = random_rhs(n, 3, seed=L)
    assert oracle.rel_err(oracle.bf_apply(bf, X), np.fft.fft(X, axis=0)) < 1e-14
    assert oracle.rel_err(oracle.bf_apply(bf, X, "C"), n * np.fft.ifft(X, axis=0)) < 1e-14


# ---------------------------------------------------------------- P5 / P6
@pytest.mark.parametrize("seed", [0, 1])
def test_P5_P6_adjoint_linearity(seed):
    bf = random_ranks_butterfly(4, [3, 5, 4, 6, 2, 7, 5, 4, 3, 3, 6, 5, 4, 4, 2, 8],
                                [4, 4, 5, 3, 6, 2, 7, 5, 3, 4, 4, 4, 5, 6, 2, 3], seed=seed,
                                rmin=1, rmax=5)
    oracle.validate(bf)
    rng = np.random.default_rng(seed)
    X = random_rhs(bf.n, 3, seed=seed + 100)
    Z = random_rhs(bf.m, 3, seed=seed + 200)
    lhs = np.vdot(Z, oracle.bf_apply(bf, X, "N"))
    rhs = np.vdot(oracle.bf_apply(bf, Z, "C"), X)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    assert not np.any(oracle.bf_apply(bf, np.zeros((bf.n, 2))))
    K = oracle.bf_dense(bf)
    np.testing.assert_allclose(oracle.bf_apply(bf, np.eye(bf.n)), K, atol=0)
    x, y = random_rhs(bf.n, 1, seed=1), random_rhs(bf.n, 1, seed=2)
    a = oracle.bf_apply(bf, 2 * x + 3 * y)
    b = 2 * oracle.bf_apply(bf, x) + 3 * oracle.bf_apply(bf, y)
    assert oracle.rel_err(a, b) < 1e-14
    T = oracle.bf_apply(bf, Z, "T")
    assert oracle.rel_err(T, np.conj(oracle.bf_apply(bf, np.conj(Z), "C"))) < 1e-15


# ---------------------------------------------------------------- P7
def _sparse_factor_product(bf):
    """K_tree as the product of the explicit factors of Eq. (3.3).

    Coefficient spaces are indexed blockwise by (l, tau, nu); each factor places its
    blocks by the stage relations of Eq. (3.2): R_{tau,nu} maps coefficient block
    (l, tau, nu) onto (l+1, 2tau, nu>>1) (top rows) and (l+1, 2tau+1, nu>>1) (bottom);
    W_{tau,nu} maps (l-1, tau>>1, 2nu) and (l-1, tau>>1, 2nu+1) onto (l, tau, nu);
    B^{lc} maps column space (lc, tau, nu) to row space (lc, tau, nu) (reading A1).
    """
    L, lc = bf.L, bf.lc

    def space(sizes):  # dict (tau, nu) -> offset, total
        off, tot = {}, 0
        for key in sorted(sizes):
            off[key] = tot
            tot += sizes[key]
        return off, tot

    def rsize(l):
        if l == L:
            return {(t, 0): bf.Ub(t).shape[1] for t in range(1 << L)}
        return {(t, v): bf.Rb(l, t, v).shape[1] for t in range(1 << l) for v in range(1 << (L - l))}

    def csize(l):
        if l == 0:
            return {(0, v): bf.Vtb(v).shape[0] for v in range(1 << L)}
        return {(t, v): bf.Wb(l, t, v).shape[0] for t in range(1 << l) for v in range(1 << (L - l))}

    # U^L : m x |row space L|
    offL, totL = space(rsize(L))
    UL = sp.lil_matrix((bf.m, totL), dtype=complex)
    for t in range(1 << L):
        r0, r1 = bf.row_leaf_ptr[t], bf.row_leaf_ptr[t + 1]
        UL[r0:r1, offL[(t, 0)]:offL[(t, 0)] + bf.Ub(t).shape[1]] = bf.Ub(t)
    prod = UL.tocsr()
    for l in range(L - 1, lc - 1, -1):
        offU, totU = space(rsize(l + 1))
        offD, totD = space(rsize(l))
        Rl = sp.lil_matrix((totU, totD), dtype=complex)
        for t in range(1 << l):
            for v in range(1 << (L - l)):
                Rb = bf.Rb(l, t, v)
                ra = rsize(l + 1)[(2 * t, v >> 1)]
                c0 = offD[(t, v)]
                a0 = offU[(2 * t, v >> 1)]
                b0 = offU[(2 * t + 1, v >> 1)]
                Rl[a0:a0 + ra, c0:c0 + Rb.shape[1]] = Rb[:ra]
                Rl[b0:b0 + Rb.shape[0] - ra, c0:c0 + Rb.shape[1]] = Rb[ra:]
        prod = prod @ Rl.tocsr()
    offR, totR = space(rsize(lc))
    offC, totC = space(csize(lc))
    Bl = sp.lil_matrix((totR, totC), dtype=complex)
    for t in range(1 << lc):
        for v in range(1 << (L - lc)):
            Bb = bf.Bb(t, v)
            Bl[offR[(t, v)]:offR[(t, v)] + Bb.shape[0], offC[(t, v)]:offC[(t, v)] + Bb.shape[1]] = Bb
    prod = prod @ Bl.tocsr()
    for l in range(lc, 0, -1):
        offU, totU = space(csize(l))
        offD, totD = space(csize(l - 1))
        Wl = sp.lil_matrix((totU, totD), dtype=complex)
        for t in range(1 << l):
            for v in range(1 << (L - l)):
                Wb = bf.Wb(l, t, v)
                ca = csize(l - 1)[(t >> 1, 2 * v)]
                r0 = offU[(t, v)]
                a0 = offD[(t >> 1, 2 * v)]
                b0 = offD[(t >> 1, 2 * v + 1)]
                Wl[r0:r0 + Wb.shape[0], a0:a0 + ca] = Wb[:, :ca]
                Wl[r0:r0 + Wb.shape[0], b0:b0 + Wb.shape[1] - ca] = Wb[:, ca:]
        prod = prod @ Wl.tocsr()
    off0, tot0 = space(csize(0))
    V0 = sp.lil_matrix((tot0, bf.n), dtype=complex)
    for v in range(1 << L):
        c0, c1 = bf.col_leaf_ptr[v], bf.col_leaf_ptr[v + 1]
        V0[off0[(0, v)]:off0[(0, v)] + bf.Vtb(v).shape[0], c0:c1] = bf.Vtb(v)
    return (prod @ V0.tocsr()).toarray()


@pytest.mark.parametrize("L,lc,seed", [(0, 0, 0), (1, 0, 1), (2, 1, 2), (3, 1, 3), (3, 2, 4),
                                       (4, 2, 5), (5, 2, 6), (5, 3, 7), (4, 0, 8), (4, 4, 9)])
def test_P7_blockwise_equals_factor_product(L, lc, seed):
    rng = np.random.default_rng(seed)
    nb = 1 << L
    bf = random_ranks_butterfly(L, rng.integers(1, 6, nb), rng.integers(1, 6, nb), seed=seed,
                                rmin=1, rmax=4, lc=lc)
    oracle.validate(bf)
    Kb = oracle.bf_dense_tree(bf)
    Kp = _sparse_factor_product(bf)
    assert np.abs(Kb - Kp).max() <= 1e-14 * max(1.0, np.abs(Kp).max())


# ---------------------------------------------------------------- P9
@pytest.mark.parametrize("kind", ["uniform", "ragged"])
def test_P9_sampled_rows_and_cols(kind):
    if kind == "uniform":
        bf = random_butterfly(L=5, leaf=4, r=3, seed=3)
        bf.row_perm = np.random.default_rng(1).permutation(bf.m)
        bf.col_perm = np.random.default_rng(2).permutation(bf.n)
    else:
        rng = np.random.default_rng(4)
        bf = random_ranks_butterfly(5, rng.integers(0, 6, 32), rng.integers(1, 6, 32), seed=4,
                                    rmin=1, rmax=5)
    X = random_rhs(bf.n, 4, seed=8)
    Z = random_rhs(bf.m, 4, seed=9)
    rows = np.random.default_rng(0).choice(bf.m, size=min(25, bf.m), replace=False)
    cols = np.random.default_rng(1).choice(bf.n, size=min(25, bf.n), replace=False)
    Y = oracle.bf_apply(bf, X)
    np.testing.assert_allclose(oracle.bf_rows_apply(bf, rows, X), Y[rows], rtol=0, atol=1e-13 * np.abs(Y).max())
    Ya = oracle.bf_apply(bf, Z, "C")
    np.testing.assert_allclose(oracle.bf_cols_apply_adj(bf, cols, Z), Ya[cols], rtol=0, atol=1e-13 * np.abs(Ya).max())


def test_P9_hodbf_sampled_rows():
    """The config-4 oracle (sampled rows of an HOD-BF, per-level bf_rows_apply on the sibling
    butterflies) equals rows of the dense HOD-BF assembly."""
    from bfinputs.configs import helmholtz_plane_hodbf
    H = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4, ncomp=2)
    X = random_rhs(H.n, 3, seed=5)
    rows = np.random.default_rng(2).choice(H.n, size=40, replace=False)
    Y = oracle.hodbf_dense(H) @ X
    np.testing.assert_allclose(oracle.hodbf_rows_apply(H, rows, X), Y[rows], rtol=0, atol=1e-13 * np.abs(Y).max())


# ---------------------------------------------------------------- P8
def _lowrank_bf_L0(Ablock):
    m, n = Ablock.shape
    return butterfly_from_blocks(0, 0, [0, m], [0, n], np.arange(m), np.arange(n),
                                 [np.eye(m)], {}, [Ablock], {}, [np.eye(n)])


def test_P8_hodbf_two_by_two_block_matrix():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
    lp = np.array([0, 4, 9])
    perm = rng.permutation(9)
    D = Stage.from_blocks([A[:4, :4], A[4:, 4:]], np.complex128)
    H = HODBF(9, 1, lp, np.arange(9), D, [[_lowrank_bf_L0(A[:4, 4:]), _lowrank_bf_L0(A[4:, :4])]])
    np.testing.assert_array_equal(oracle.hodbf_dense(H), A)
    H.perm = perm
    Ad = np.zeros_like(A)
    Ad[np.ix_(perm, perm)] = A
    np.testing.assert_array_equal(oracle.hodbf_dense(H), Ad)
    X = random_rhs(9, 3, seed=1)
    for op in "NCT":
        assert oracle.rel_err(oracle.hodbf_apply(H, X, op), oracle.apply_op(Ad, X, op)) < 1e-15


def test_hodbf_extract_two_by_two_block_matrix():
    """extract_HODBF of the L_H = 1 HOD-BF whose blocks are an arbitrary 2x2 block matrix (P8):
    exactly the entries of that matrix, under a permutation, repeats included."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
    lp = np.array([0, 4, 9])
    perm = rng.permutation(9)
    D = Stage.from_blocks([A[:4, :4], A[4:, 4:]], np.complex128)
    H = HODBF(9, 1, lp, perm, D, [[_lowrank_bf_L0(A[:4, 4:]), _lowrank_bf_L0(A[4:, :4])]])
    Ad = np.zeros_like(A)
    Ad[np.ix_(perm, perm)] = A
    I, J = rng.integers(0, 9, 7), rng.integers(0, 9, 5)
    np.testing.assert_array_equal(oracle.hodbf_extract(H, I, J), Ad[np.ix_(I, J)])


def test_P8_hodbf_zero_offdiag_is_blockdiag():
    rng = np.random.default_rng(1)
    LH, leaf = 3, 3
    n = leaf << LH
    lp = np.arange((1 << LH) + 1) * leaf
    Ds = [rng.standard_normal((leaf, leaf)) + 0j for _ in range(1 << LH)]
    off = []
    for l in range(1, LH + 1):
        sz = leaf << (LH - l)
        off.append([_lowrank_bf_L0(np.zeros((sz, sz))) for _ in range(1 << l)])
    H = HODBF(n, LH, lp, np.arange(n), Stage.from_blocks(Ds, np.complex128), off)
    import scipy.linalg as sla
    np.testing.assert_array_equal(oracle.hodbf_dense(H), sla.block_diag(*Ds))


# ---------------------------------------------------------------- ID building block
def test_ID_exact_on_low_rank():
    rng = np.random.default_rng(2)
    M = (rng.standard_normal((40, 6)) + 1j * rng.standard_normal((40, 6))) @ \
        (rng.standard_normal((6, 30)) + 1j * rng.standard_normal((6, 30)))
    U, I = row_id(M, 1e-12)
    assert U.shape[1] == 6
    np.testing.assert_allclose(U[I], np.eye(6), atol=0)
    assert np.linalg.norm(U @ M[I] - M) < 1e-11 * np.linalg.norm(M)
    Vt, J = col_id(M, 1e-12)
    assert Vt.shape[0] == 6
    np.testing.assert_allclose(Vt[:, J], np.eye(6), atol=0)
    assert np.linalg.norm(M[:, J] @ Vt - M) < 1e-11 * np.linalg.norm(M)


# ------------------------------------------------------------------ extraction (NEXT-1)
@pytest.mark.parametrize("L,m0", [(4, 2), (3, 3)])
def test_extract_identity_closed_form(L, m0):
    """extract_BF of the closed-form identity butterfly (P1) is the Kronecker delta of the
    requested indices (repeats included)."""
    bf = identity_butterfly(L, m0)
    rng = np.random.default_rng(L)
    I = rng.integers(0, bf.m, 9)
    J = np.concatenate([I[:4], rng.integers(0, bf.n, 5)])
    E = oracle.bf_extract(bf, I, J)
    assert np.array_equal(E, (I[:, None] == J[None, :]).astype(np.complex128))


def test_extract_dft_closed_form():
    """extract_BF of the closed-form DFT butterfly (P3) is omega^(i j), omega = e^(-2 pi i / n)."""
    L = 8
    bf = dft_butterfly(L)
    n = bf.n
    rng = np.random.default_rng(3)
    I, J = rng.integers(0, n, 11), rng.integers(0, n, 7)
    ref = np.exp(-2j * np.pi * ((I[:, None] * J[None, :]) % n) / n)
    assert np.abs(oracle.bf_extract(bf, I, J) - ref).max() < 1e-13
