"""GPU parity of bf_extract (Alg. 3 extract_BF; the sub-matrix
K(I, J) as a partial matvec over the touched blocks) against the CPU oracle's entries of K:
random uniform-rank butterflies (fused-path shapes; extraction runs the generic kernel),
ragged ranks, permuted rows / columns, repeated and scattered indices, single entries, whole
leaf blocks, both dtypes; the closed-form identity extracts exactly."""
import numpy as np
import pytest

import oracle
from bfinputs import identity_butterfly, random_butterfly, random_ranks_butterfly
import paper_2007_00202_b200 as pkg

pytestmark = pytest.mark.gpu

TOL = {np.complex128: 1e-12, np.complex64: 1e-5}


def _get(h, I, J):
    return h.extract(I, J).cpu().numpy()


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,leaf,r", [(6, 16, 16), (9, 16, 16), (5, 32, 8)])
def test_extract_random(L, leaf, r, dtype):
    bf = random_butterfly(L=L, leaf=leaf, r=r, seed=L + r, dtype=dtype)
    rng = np.random.default_rng(L)
    bf.row_perm = rng.permutation(bf.m).astype(np.int64)
    bf.col_perm = rng.permutation(bf.n).astype(np.int64)
    h = pkg.BFHandle(bf)
    cases = [
        (rng.integers(0, bf.m, 37), rng.integers(0, bf.n, 29)),          # scattered, repeats
        (np.arange(leaf, 3 * leaf), np.arange(bf.n - 2 * leaf, bf.n)),    # contiguous user ranges
        ([5], [bf.n - 1]),                                                # one entry
        (rng.integers(0, bf.m, 300), rng.integers(0, bf.n, 70)),         # many leaves
    ]
    for I, J in cases:
        got = _get(h, I, J)
        ref = oracle.bf_extract(bf, I, J)
        assert got.shape == (len(I), len(J))
        assert oracle.rel_err(got, ref) <= TOL[dtype], (len(I), len(J))


def test_extract_ragged_ranks():
    rng = np.random.default_rng(4)
    bf = random_ranks_butterfly(6, rng.integers(1, 9, 64), rng.integers(1, 9, 64), seed=4, rmin=1, rmax=7)
    h = pkg.BFHandle(bf)
    I, J = rng.integers(0, bf.m, 41), rng.integers(0, bf.n, 23)
    assert oracle.rel_err(_get(h, I, J), oracle.bf_extract(bf, I, J)) <= 1e-12


def test_extract_identity_exact():
    bf = identity_butterfly(6, 4)
    h = pkg.BFHandle(bf)
    rng = np.random.default_rng(1)
    I = rng.integers(0, bf.m, 50)
    J = np.concatenate([I[:20], rng.integers(0, bf.n, 30)])
    np.testing.assert_array_equal(_get(h, I, J), (I[:, None] == J[None, :]).astype(np.complex128))


def test_extract_errors():
    bf = random_butterfly(L=3, leaf=8, r=4, seed=2)
    h = pkg.BFHandle(bf)
    with pytest.raises(pkg.BFError):
        h.extract([bf.m], [0])
    with pytest.raises(pkg.BFError):
        h.extract([0], [-1])
    assert h.extract([], [1, 2]).shape == (0, 2)


# ------------------------------------------------------------------ extract_HODBF
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_hodbf_extract(dtype):
    """hodbf_extract: dense-leaf entries plus, for every other entry, the sibling
    butterfly of the level where its row's and column's nodes split."""
    from bfinputs.configs import helmholtz_plane_hodbf
    H = helmholtz_plane_hodbf(32, 16, 10.0, 1e-4).astype(dtype)
    h = pkg.HODBFHandle(H)
    rng = np.random.default_rng(2)
    t = H.perm[int(H.leaf_ptr[5]):int(H.leaf_ptr[6])]  # the user indices of one leaf
    cases = [
        (rng.integers(0, H.n, 57), rng.integers(0, H.n, 33)),   # scattered, every level, repeats
        (t, t),                                                  # one dense leaf block
        (t, H.perm[int(H.leaf_ptr[40]):int(H.leaf_ptr[44])]),   # a far off-diagonal block
        ([3], [H.n - 1]),
    ]
    for I, J in cases:
        got = h.extract(I, J).cpu().numpy()
        assert oracle.rel_err(got, oracle.hodbf_extract(H, I, J)) <= TOL[dtype], (len(I), len(J))


@pytest.mark.parametrize("L,lc", [(0, 0), (5, 0), (5, 5), (4, 1)])
def test_extract_centre_edge_cases(L, lc):
    """lc at 0 or L (no W or no R stages), and L = 0 (K = U B Vt: one dense block)."""
    bf = random_butterfly(L=L, leaf=16, r=8, seed=3 + L + lc, lc=lc)
    h = pkg.BFHandle(bf)
    rng = np.random.default_rng(L + lc)
    I, J = rng.integers(0, bf.m, 23), rng.integers(0, bf.n, 17)
    assert oracle.rel_err(_get(h, I, J), oracle.bf_extract(bf, I, J)) <= 1e-12


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_extract_list(dtype):
    """Alg. 3's list form (bf_extract_list): several (I, J) requests in one batched evaluation --
    scattered, repeated, overlapping, single entries, empty ones -- each equals the oracle's entries
    and the single-request bf_extract."""
    bf = random_butterfly(L=7, leaf=16, r=16, seed=3, dtype=dtype)
    rng = np.random.default_rng(7)
    bf.row_perm = rng.permutation(bf.m).astype(np.int64)
    bf.col_perm = rng.permutation(bf.n).astype(np.int64)
    h = pkg.BFHandle(bf)
    pairs = [(rng.integers(0, bf.m, 20), rng.integers(0, bf.n, 33)),
             (np.arange(40, 90), np.arange(0, 16)),
             ([3], [bf.n - 2]),
             (rng.integers(0, bf.m, 20), rng.integers(0, bf.n, 33)),
             ([], [1, 2]),
             (np.arange(0, 16), rng.integers(0, bf.n, 200))]
    got = h.extract_list(pairs)
    for (I, J), G in zip(pairs, got):
        assert G.shape == (len(I), len(J))
        if len(I) == 0:
            continue
        ref = oracle.bf_extract(bf, I, J)
        assert oracle.rel_err(G.cpu().numpy(), ref) <= TOL[dtype]
        assert oracle.rel_err(G.cpu().numpy(), _get(h, I, J)) <= TOL[dtype]
