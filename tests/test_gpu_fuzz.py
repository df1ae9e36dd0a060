"""Seeded randomised parity sweep: many small butterflies drawn across the shape space the
library dispatches on -- the fused kernels (uniform rank 16 and ranks <= 16 padded to 16, leaves
16-256, every window depth), the generic kernels (ragged ranks up to 40, uneven leaves, rank-0
blocks), random row / column permutations, non-canonical block orderings (level_maps), every
op, both dtypes, and nrhs across the kernels' column regimes (1-8 narrow, 9-16 one column half,
17-32, several 32-column tiles with a ragged tail) -- each against the dense definition
(oracle.bf_dense, Eq. 3.1-3.2).  Bar: BASELINE.json's 1e-12 (complex128) / 1e-5 (complex64)."""
import numpy as np
import pytest
import torch

import oracle
from bfinputs import random_butterfly, random_level_maps, random_ranks_butterfly, random_rhs, slot_ordered
import paper_2007_00202_b200 as pkg

pytestmark = pytest.mark.gpu

TOL = {np.complex128: 1e-12, np.complex64: 1e-5}
NRHS = [1, 3, 8, 9, 13, 16, 17, 31, 32, 33, 47, 64, 70]


def _case(seed):
    """One random butterfly, its level maps (or None) and the launch regime it should take."""
    rng = np.random.default_rng(1000 + seed)
    dtype = np.complex128 if rng.random() < 0.6 else np.complex64
    kind = rng.choice(["fast16", "padded", "ragged"], p=[0.35, 0.25, 0.4])
    if kind == "fast16":
        L = int(rng.integers(1, 8))  # n = leaf 2^L <= 4096 (the dense oracle)
        leaf = int(rng.choice([16, 32, 64, 128, 256][: max(1, min(5, 9 - L))]))
        bf = random_butterfly(L=L, leaf=leaf, r=16, seed=seed, dtype=dtype, lc=int(rng.integers(0, L + 1)))
    else:
        L = int(rng.integers(0, 7))
        nb = 1 << L
        if kind == "padded" and L >= 1:
            leaf = int(rng.choice([16, 32, 64]))
            rows = cols = np.full(nb, leaf)
            rmin, rmax = int(rng.integers(0, 4)), int(rng.integers(4, 17))
        else:
            kind = "ragged"
            rows, cols = rng.integers(0, 40, nb), rng.integers(1, 40, nb)
            rmin, rmax = int(rng.integers(0, 3)), int(rng.integers(3, 41))
        bf = random_ranks_butterfly(L, rows, cols, seed=seed, rmin=rmin, rmax=rmax,
                                    lc=int(rng.integers(0, L + 1)), dtype=dtype)
    if rng.random() < 0.5:
        bf.row_perm = rng.permutation(bf.m).astype(np.int64)
        bf.col_perm = rng.permutation(bf.n).astype(np.int64)
    maps = random_level_maps(bf.L, seed=seed) if rng.random() < 0.3 else None
    return bf, maps, dtype, kind, rng


@pytest.mark.parametrize("seed", range(160))
def test_fuzz_apply(seed):
    bf, maps, dtype, kind, rng = _case(seed)
    h = pkg.BFHandle(slot_ordered(bf, maps) if maps is not None else bf, level_maps=maps)
    if kind in ("fast16", "padded") and bf.L >= 1:
        # (selection-only factors would stay generic; random Gaussian factors never are)
        assert h.rounds("N")[0]["name"].startswith("k_leaf"), (kind, bf.L)
    K = oracle.bf_dense(bf)
    for op in ("N", "C", "T"):
        nr = int(rng.choice(NRHS))
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=seed + 17, dtype=dtype)
        Y = h.apply(torch.from_numpy(np.ascontiguousarray(X.T)).cuda(), op)
        torch.cuda.synchronize()
        err = oracle.rel_err(Y.cpu().numpy().T, oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (seed, kind, bf.L, op, nr, err)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_hodbf(seed):
    """HOD-BF applies on Helmholtz planes of random size, compression tolerance, nrhs and op,
    both dtypes, against the assembled dense matrix."""
    from bfinputs.configs import helmholtz_plane_hodbf
    rng = np.random.default_rng(5000 + seed)
    nx, ny = int(rng.integers(6, 25)), int(rng.integers(6, 25))
    tol = float(rng.choice([1e-4, 1e-6, 1e-8]))
    H = helmholtz_plane_hodbf(nx, ny, 10.0, tol)
    dtype = np.complex64 if seed % 3 == 2 else np.complex128
    if dtype == np.complex64:
        H = H.astype(np.complex64)
    h = pkg.HODBFHandle(H)
    A = oracle.hodbf_dense(H)
    for op in ("N", "C", "T"):
        nr = int(rng.choice(NRHS))
        X = random_rhs(H.n, nr, seed=seed + 3, dtype=dtype)
        Y = h.apply(torch.from_numpy(np.ascontiguousarray(X.T)).cuda(), op)
        torch.cuda.synchronize()
        err = oracle.rel_err(Y.cpu().numpy().T, oracle.apply_op(A, X, op))
        assert err <= TOL[dtype], (seed, nx, ny, tol, op, nr, err)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_extract(seed):
    """bf_extract / bf_extract_list (Alg. 3) on random butterflies: random lists of scattered
    (rows, cols) requests (duplicates and empty requests included) against the dense gather."""
    bf, maps, dtype, kind, rng = _case(10_000 + seed)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    pairs = []
    for _ in range(int(rng.integers(1, 5))):
        nI, nJ = int(rng.integers(0, min(bf.m, 70) + 1)), int(rng.integers(0, min(bf.n, 70) + 1))
        pairs.append((rng.integers(0, max(bf.m, 1), nI), rng.integers(0, max(bf.n, 1), nJ)))
    outs = h.extract_list(pairs)
    torch.cuda.synchronize()
    for (I, J), E in zip(pairs, outs):
        ref = K[np.ix_(I, J)]
        if ref.size:
            assert oracle.rel_err(E.cpu().numpy(), ref) <= TOL[dtype], (seed, kind, len(I), len(J))
    I, J = pairs[0]
    if len(I) and len(J):
        assert oracle.rel_err(h.extract(I, J).cpu().numpy(), K[np.ix_(I, J)]) <= TOL[dtype]


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_split_emulated(seed):
    """The multi-GPU split (bf_dist_*) on random shapes and rank counts, the P rank-local plans run
    in turn on one device with the exchange replayed as copies (tests/test_gpu_dist.emulate)."""
    from test_gpu_dist import _subtree_perm, emulate
    rng = np.random.default_rng(20_000 + seed)
    dtype = np.complex128 if seed % 4 else np.complex64
    P = int(rng.choice([2, 4, 8]))
    p = P.bit_length() - 1
    L = int(rng.integers(2 * p, 9))
    lc = int(rng.integers(p, L - p + 1))
    if seed % 2:
        bf = random_butterfly(L=L, leaf=16, r=16, seed=seed, dtype=dtype, lc=lc)
    else:
        nb = 1 << L
        bf = random_ranks_butterfly(L, rng.integers(0, 9, nb), rng.integers(1, 9, nb), seed=seed, rmin=1,
                                    rmax=int(rng.integers(2, 12)), lc=lc, dtype=dtype)
    bf.row_perm = _subtree_perm(bf.m, bf.row_leaf_ptr, bf.L, p, seed)
    bf.col_perm = _subtree_perm(bf.n, bf.col_leaf_ptr, bf.L, p, seed + 1)
    K = oracle.bf_dense(bf)
    for op in ("N", "C", "T"):
        nr = int(rng.choice(NRHS))
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=seed + 5, dtype=dtype)
        err = oracle.rel_err(emulate(bf, X, op, P), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (seed, P, L, lc, op, nr, err)
