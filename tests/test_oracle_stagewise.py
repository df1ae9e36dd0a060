"""Pins of the level-by-level CPU oracle (oracle/stagewise.py), of the
HOD-BF oracle at depth (L_H >= 3) and negative cases of oracle.validate.  No GPU.

The stagewise apply shares no code with oracle/dense.py; here it is pinned
  * against the blockwise dense definition Eq. (3.1)-(3.2) (oracle.bf_dense) on ragged ranks,
    uneven leaves, odd L and every lc, in both the per-block and the batched form;
  * against closed forms that involve neither oracle: the DFT butterfly (P3) vs numpy.fft at
    L up to 16, the identity butterfly (P1) exactly;
  * by the dot-product identity <K X, Z> = <X, K^H Z> (P5).
"""
import numpy as np
import pytest

import oracle
from oracle.stagewise import bf_apply_stagewise, hodbf_apply_stagewise
from bfinputs import (Stage, bitrev, butterfly_from_blocks, dft_butterfly, identity_butterfly,
                      random_butterfly, random_ranks_butterfly, random_rhs)
from bfinputs.factors import HODBF


@pytest.mark.parametrize("L", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("seed", [0, 1])
def test_stagewise_ragged_every_lc(L, seed):
    """Ragged ranks (including rank 0), uneven and empty leaves, random perms, every lc."""
    rng = np.random.default_rng(100 * L + seed)
    nb = 1 << L
    rows = rng.integers(0, 7, nb)
    cols = rng.integers(1, 7, nb)
    for lc in range(L + 1):
        bf = random_ranks_butterfly(L, rows, cols, seed=seed + 10 * lc, rmin=0 if seed else 1, rmax=5, lc=lc)
        K = oracle.bf_dense(bf)
        X = random_rhs(bf.n, 3, seed=lc)
        Z = random_rhs(bf.m, 3, seed=lc + 50)
        for op, V in (("N", X), ("C", Z), ("T", Z)):
            ref = oracle.apply_op(K, V, op)
            got = bf_apply_stagewise(bf, V, op)
            assert oracle.rel_err(got, ref) < 1e-14, (L, lc, op)


@pytest.mark.parametrize("L,lc", [(3, 0), (3, 1), (4, 2), (5, 2), (5, 5), (6, 3)])
@pytest.mark.parametrize("batched", [True, False])
def test_stagewise_uniform_batched_and_blocks(L, lc, batched):
    """The batched (stacked-block) form and the per-block form both equal the dense definition
    on a uniform butterfly with non-square blocks (leaf 5, rank 3) and random perms."""
    bf = random_butterfly(L=L, leaf=5, r=3, seed=L + lc, lc=lc)
    bf.row_perm = np.random.default_rng(1).permutation(bf.m)
    bf.col_perm = np.random.default_rng(2).permutation(bf.n)
    K = oracle.bf_dense(bf)
    X = random_rhs(bf.n, 4, seed=3)
    for op in "NCT":
        got = bf_apply_stagewise(bf, X, op, threads=3, batched=batched)
        assert oracle.rel_err(got, oracle.apply_op(K, X, op)) < 1e-14, op


@pytest.mark.parametrize("L", [6, 11, 16])
def test_stagewise_dft_vs_numpy_fft(L):
    """P3 without the dense oracle: the closed-form DFT butterfly applied stage by stage equals
    numpy.fft.fft (op N) and n * ifft (op C)."""
    bf = dft_butterfly(L)
    X = random_rhs(bf.n, 3, seed=L)
    assert oracle.rel_err(bf_apply_stagewise(bf, X, "N"), np.fft.fft(X, axis=0)) < 1e-14 * L
    assert oracle.rel_err(bf_apply_stagewise(bf, X, "C"), bf.n * np.fft.ifft(X, axis=0)) < 1e-14 * L
    # batched and per-block forms agree on this uniform (rank 1, leaf 1) case
    if L <= 11:
        assert oracle.rel_err(bf_apply_stagewise(bf, X, "N", batched=False), np.fft.fft(X, axis=0)) < 1e-14 * L


@pytest.mark.parametrize("L,m0", [(3, 1), (4, 2), (5, 3), (6, 16)])
def test_stagewise_identity_exact(L, m0):
    """P1: the selection factors of the identity butterfly reproduce X exactly, both forms."""
    bf = identity_butterfly(L, m0)
    X = random_rhs(bf.n, 5, seed=L)
    for batched in (True, False):
        np.testing.assert_array_equal(bf_apply_stagewise(bf, X, "N", batched=batched), X)
        np.testing.assert_array_equal(bf_apply_stagewise(bf, X, "C", batched=batched), X)


def test_stagewise_dot_product_cfg5_shape():
    """P5 on the config-5 shape at L = 8 (leaf 64, rank 16): <K X, Z> = <X, K^H Z>, and the
    per-block form equals the batched one."""
    bf = random_butterfly(L=8, leaf=64, r=16, seed=1)
    X = random_rhs(bf.n, 6, seed=11)
    Z = random_rhs(bf.m, 6, seed=12)
    Y = bf_apply_stagewise(bf, X, "N")
    Ya = bf_apply_stagewise(bf, Z, "C")
    lhs, rhs = np.vdot(Z, Y), np.vdot(Ya, X)
    assert abs(lhs - rhs) < 1e-13 * np.linalg.norm(Z) * np.linalg.norm(Y)
    assert oracle.rel_err(bf_apply_stagewise(bf, X, "N", batched=False), Y) < 1e-14


# ---------------------------------------------------------------- HOD-BF at depth
def _L0_bf(A):
    m, n = A.shape
    return butterfly_from_blocks(0, 0, [0, m], [0, n], np.arange(m), np.arange(n),
                                 [np.eye(m)], {}, [A], {}, [np.eye(n)])


def _dense_hodbf(LH, leaf_sizes, seed):
    """An HOD-BF whose every block is an arbitrary dense matrix (off-diagonals as L = 0
    butterflies, P8): it must reproduce that matrix exactly, at any depth."""
    rng = np.random.default_rng(seed)
    lp = np.concatenate([[0], np.cumsum(leaf_sizes)]).astype(np.int64)
    n = int(lp[-1])
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    D = Stage.from_blocks([A[lp[t]:lp[t + 1], lp[t]:lp[t + 1]] for t in range(1 << LH)], np.complex128)
    off = []
    for l in range(1, LH + 1):
        w = 1 << (LH - l)
        lev = []
        for tau in range(1 << l):
            r0, r1 = lp[tau * w], lp[(tau + 1) * w]
            s = tau ^ 1
            c0, c1 = lp[s * w], lp[(s + 1) * w]
            lev.append(_L0_bf(A[r0:r1, c0:c1]))
        off.append(lev)
    perm = rng.permutation(n).astype(np.int64)
    H = HODBF(n, LH, lp, perm, D, off)
    Au = np.zeros_like(A)
    Au[np.ix_(perm, perm)] = A
    return H, Au


@pytest.mark.parametrize("LH,seed", [(3, 0), (4, 1), (5, 2)])
def test_P8_hodbf_dense_blocks_at_depth(LH, seed):
    """P8 at L_H >= 3: every block of a known matrix placed in the HOD-BF format; the dense
    assembly, the block-by-block oracle apply and the stagewise apply all reproduce it."""
    sizes = np.random.default_rng(seed).integers(1, 5, 1 << LH)
    H, A = _dense_hodbf(LH, sizes, seed)
    np.testing.assert_allclose(oracle.hodbf_dense(H), A, rtol=0, atol=0)
    X = random_rhs(H.n, 4, seed=seed)
    for op in "NCT":
        ref = oracle.apply_op(A, X, op)
        assert oracle.rel_err(oracle.hodbf_apply(H, X, op), ref) < 1e-15, op
        assert oracle.rel_err(hodbf_apply_stagewise(H, X, op), ref) < 1e-15, op


def _dft_hodbf(LH, seed):
    """HOD-BF with leaf 1 whose level-l off-diagonal blocks are closed-form DFT butterflies of
    L_B = LH - l levels (P3): A(T_tau, T_{tau^1}) = F_{2^(LH-l)} exactly, so the assembled
    matrix is known in closed form and the butterflies have real depth."""
    rng = np.random.default_rng(seed)
    n = 1 << LH
    lp = np.arange(n + 1, dtype=np.int64)
    d = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    D = Stage.from_blocks([np.array([[v]]) for v in d], np.complex128)
    A = np.diag(d)
    off = []
    for l in range(1, LH + 1):
        sz = 1 << (LH - l)
        bfs = []
        for tau in range(1 << l):
            # HOD-BF off-diagonal butterflies are tree-local (identity perms): in tree order the
            # DFT butterfly is F with rows and columns bit-reversed, F_tree[i, j] = w^(rev(i) rev(j))
            bft = dft_butterfly(LH - l)
            bft.row_perm = np.arange(sz, dtype=np.int64)
            bft.col_perm = np.arange(sz, dtype=np.int64)
            bfs.append(bft)
            r0, s = tau * sz, (tau ^ 1) * sz
            j = bitrev(np.arange(sz), LH - l)
            A[r0:r0 + sz, s:s + sz] = np.exp(-2j * np.pi * (np.outer(j, j) % sz) / sz)
        off.append(bfs)
    return HODBF(n, LH, lp, np.arange(n), D, off), A


@pytest.mark.parametrize("LH", [3, 5])
def test_P8_P3_hodbf_dft_offdiagonals(LH):
    """HOD-BF with DFT-butterfly off-diagonals at every level (depth L_B = L_H - l): the dense
    assembly, the oracle apply and the stagewise apply equal the closed-form matrix."""
    H, A = _dft_hodbf(LH, LH)
    assert np.abs(oracle.hodbf_dense(H) - A).max() < 1e-13
    X = random_rhs(H.n, 3, seed=LH)
    for op in "NCT":
        ref = oracle.apply_op(A, X, op)
        assert oracle.rel_err(oracle.hodbf_apply(H, X, op), ref) < 1e-14, op
        assert oracle.rel_err(hodbf_apply_stagewise(H, X, op), ref) < 1e-14, op


def test_hodbf_stagewise_vs_dense_helmholtz():
    """A constructed (ID-compressed, ragged ranks) Helmholtz HOD-BF with L_H = 4: stagewise
    apply == dense assembly times X, ops N / C / T."""
    from bfinputs.configs import helmholtz_plane_hodbf
    H = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4)
    assert H.LH >= 3
    A = oracle.hodbf_dense(H)
    X = random_rhs(H.n, 5, seed=2)
    for op in "NCT":
        ref = oracle.apply_op(A, X, op)
        assert oracle.rel_err(hodbf_apply_stagewise(H, X, op), ref) < 1e-14, op
        assert oracle.rel_err(oracle.hodbf_apply(H, X, op), ref) < 1e-14, op


# ---------------------------------------------------------------- validate: negative cases
def _bad(kind):
    bf = random_ranks_butterfly(3, [2, 3, 1, 4, 2, 2, 3, 1], [1, 2, 3, 2, 1, 2, 2, 3], seed=5, rmin=1, rmax=4)
    if kind == "leaf_ptr_sum":
        bf.row_leaf_ptr = bf.row_leaf_ptr.copy()
        bf.row_leaf_ptr[-1] += 1
    elif kind == "leaf_ptr_monotone":
        bf.col_leaf_ptr = bf.col_leaf_ptr.copy()
        bf.col_leaf_ptr[2], bf.col_leaf_ptr[3] = bf.col_leaf_ptr[3] + 1, bf.col_leaf_ptr[2]
    elif kind == "perm":
        bf.row_perm = bf.row_perm.copy()
        bf.row_perm[0] = bf.row_perm[1]
    elif kind == "lc":
        bf.lc = bf.L + 1
    elif kind == "R_chain":
        st = bf.R[0]
        blocks = [st.block(i) for i in range(st.nblocks)]
        blocks[3] = np.vstack([blocks[3], np.zeros((1, blocks[3].shape[1]))])
        bf.R[0] = Stage.from_blocks(blocks, np.complex128)
    elif kind == "W_chain":
        st = bf.W[0]
        blocks = [st.block(i) for i in range(st.nblocks)]
        blocks[1] = np.hstack([blocks[1], np.zeros((blocks[1].shape[0], 1))])
        bf.W[0] = Stage.from_blocks(blocks, np.complex128)
    elif kind == "B_shape":
        st = bf.B
        blocks = [st.block(i) for i in range(st.nblocks)]
        blocks[5] = np.zeros((blocks[5].shape[0] + 1, blocks[5].shape[1]))
        bf.B = Stage.from_blocks(blocks, np.complex128)
    elif kind == "U_rows":
        st = bf.U
        blocks = [st.block(i) for i in range(st.nblocks)]
        blocks[2] = np.zeros((blocks[2].shape[0] + 1, blocks[2].shape[1]))
        bf.U = Stage.from_blocks(blocks, np.complex128)
    return bf


def test_validate_accepts_good():
    oracle.validate(_bad("none"))


@pytest.mark.parametrize("kind", ["leaf_ptr_sum", "leaf_ptr_monotone", "perm", "lc", "R_chain", "W_chain",
                                  "B_shape", "U_rows"])
def test_validate_rejects(kind):
    with pytest.raises(AssertionError):
        oracle.validate(_bad(kind))
