"""GPU parity of the fused window-pass path (uniform rank 16, leaves multiple of 16)
against the CPU oracle: every pass layout (L = 1..9, odd / even L, all lc), op N / C / T,
permuted rows and columns, ragged nrhs, and config 5 full-vector agreement with the
generic batched path."""
import numpy as np
import pytest
import torch

import oracle
from bfinputs import random_butterfly, random_ranks_butterfly, random_rhs
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
    names = [r["name"] for r in h.rounds("N")]
    # leaf-in launch, window passes (complex128: the last one runs the fused row-leaf op),
    # leaf-out launch (complex64)
    fused = dtype == np.complex128
    assert names[0].startswith("k_leaf") and names[-1].startswith("k_bf_pass" if fused else "k_leaf"), names
    assert all(n.startswith("k_bf_pass") for n in names[1:len(names) - (0 if fused else 1)]), names
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 32), ("C", 45), ("T", 7)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=L + nr, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,leaf,lc,rmin,rmax", [(5, 32, None, 0, 16), (4, 16, 1, 1, 9), (6, 64, 4, 5, 16),
                                                 (3, 128, 0, 0, 12), (5, 32, 5, 8, 8), (7, 16, None, 2, 15)])
@pytest.mark.parametrize("nrhs", [1, 16, 40])
def test_fast_ragged_ranks_padded(L, leaf, lc, rmin, rmax, nrhs, dtype):
    """Ragged ranks <= 16 (rank-0 blocks included) on uniform power-of-two leaves run on the
    fused kernels with every block zero-padded to rank 16 at create (pad_rank16; VERDICT r1 item
    6): the fused launch sequence, ops N / C / T against the dense definition."""
    nb = 1 << L
    bf = random_ranks_butterfly(L, np.full(nb, leaf), np.full(nb, leaf), seed=31 * L + rmax, rmin=rmin, rmax=rmax,
                                lc=lc, dtype=dtype)
    rng = np.random.default_rng(L + rmax)
    bf.row_perm = rng.permutation(bf.m).astype(np.int64)
    bf.col_perm = rng.permutation(bf.n).astype(np.int64)
    h = pkg.BFHandle(bf)
    assert h.rounds("N")[0]["name"].startswith("k_leaf"), "expected the fused path"
    K = oracle.bf_dense(bf)
    for op in "NCT":
        X = random_rhs(bf.n if op == "N" else bf.m, nrhs, seed=L + nrhs, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,leaf", [(2, 256), (3, 128), (4, 256), (8, 16)])
@pytest.mark.parametrize("nrhs", [1, 33])
def test_fast_large_leaves_and_thin_blocks(L, leaf, nrhs, dtype):
    """The largest fast-path leaves (128, 256: several chunks per leaf item in both leaf
    kernels), a single right-hand side and one column past a tile boundary."""
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=7 * L + leaf, dtype=dtype)
    h = pkg.BFHandle(bf)
    assert h.rounds("N")[0]["name"].startswith("k_leaf"), "expected the fused path"
    K = oracle.bf_dense(bf)
    for op in "NCT":
        X = random_rhs(bf.n if op == "N" else bf.m, nrhs, seed=L + nrhs, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,leaf,lc", [(3, 16, None), (4, 32, None), (6, 16, 1), (7, 16, None), (5, 64, 5),
                                       (3, 256, None)])
@pytest.mark.parametrize("nrhs", [9, 12, 16])
def test_fast_half_tile_nrhs(L, leaf, lc, nrhs, dtype):
    """9 <= nrhs <= 16 selects separate instantiations: the pass kernel with one working column
    half (HV = 1: the second half's warps exit, release counts cover the first half only) and
    the 16-column leaf kernels (PolC*<2>).  Every pass layout, permuted rows and columns, op
    N / C / T."""
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=L * 10 + leaf + nrhs, lc=lc, dtype=dtype)
    rng = np.random.default_rng(L + nrhs)
    bf.row_perm = rng.permutation(bf.m).astype(np.int64)
    bf.col_perm = rng.permutation(bf.n).astype(np.int64)
    h = pkg.BFHandle(bf)
    assert h.rounds("N")[0]["name"].startswith("k_leaf"), "expected the fused path"
    K = oracle.bf_dense(bf)
    for op in "NCT":
        X = random_rhs(bf.n if op == "N" else bf.m, nrhs, seed=L + nrhs, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, nrhs, err)


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
    assert hg.rounds("N")[0]["name"].startswith("k_stage_tile")
    Yg = hg.apply(Xd)
    Yga = hg.apply(Xd, "C")
    torch.cuda.synchronize()
    tol = 1e-13 if dtype == np.complex128 else 1e-5
    assert (torch.linalg.norm(Yf - Yg) / torch.linalg.norm(Yg)).item() <= tol
    assert (torch.linalg.norm(Yfa - Yga) / torch.linalg.norm(Yga)).item() <= tol


def leaf_block_perm(n, leaf, seed):
    """A permutation that moves whole leaves: every leaf is a contiguous run of user rows (the
    leaf kernels then move X / Y with TMA tiles instead of per-row gathers)."""
    rng = np.random.default_rng(seed)
    blocks = rng.permutation(n // leaf)
    return (blocks[:, None] * leaf + np.arange(leaf)[None, :]).reshape(-1).astype(np.int64)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("L,leaf,perm", [(3, 16, "id"), (5, 64, "block"), (4, 32, "block"), (7, 16, "id"),
                                         (2, 128, "block"), (3, 256, "id"), (6, 64, "block")])
def test_fast_contiguous_leaves(L, leaf, perm, dtype):
    """Contiguous leaves (identity or leaf-block permutations): X read by 2-D TMA tiles, Y written
    by row runs; ragged nrhs (out-of-bounds TMA columns are zero-filled), op N / C / T."""
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=L + leaf, dtype=dtype)
    if perm == "block":
        bf.row_perm = leaf_block_perm(bf.m, leaf, 1)
        bf.col_perm = leaf_block_perm(bf.n, leaf, 2)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 32), ("C", 45), ("T", 7), ("N", 70)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=L + nr, dtype=dtype)
        err = oracle.rel_err(host(h.apply(dev(X), op)), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, nr, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("pad", [1, 2, 16])
def test_fast_padded_ld(pad, dtype):
    """X and Y as column blocks of wider buffers (ld > rows): TMA when ld * sizeof is a multiple
    of 16 bytes, the gather path otherwise (odd ld for complex64)."""
    bf = random_butterfly(L=5, leaf=32, r=16, seed=pad, dtype=dtype)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    nr = 40
    X = random_rhs(bf.n, nr, seed=pad, dtype=dtype)
    big = torch.zeros((nr, bf.n + pad), dtype=dev(X).dtype, device="cuda")
    big[:, :bf.n] = dev(X)
    outb = torch.full((nr, bf.m + pad), 7.0, dtype=big.dtype, device="cuda")
    Y = h.apply(big[:, :bf.n], "N", out=outb[:, :bf.m])
    err = oracle.rel_err(host(Y), K @ X)
    assert err <= TOL[dtype], err
    assert torch.all(outb[:, bf.m:] == 7.0), "wrote outside the Y block"


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_fast_tma_equals_gather(monkeypatch, dtype):
    """The TMA tile path and the per-row gather path of the leaf kernels agree bit for bit
    (same arithmetic, same order; only the data movement differs)."""
    bf = random_butterfly(L=6, leaf=64, r=16, seed=3, dtype=dtype)
    X = dev(random_rhs(bf.n, 50, seed=4, dtype=dtype))
    h = pkg.BFHandle(bf)
    Y1, Y1c = h.apply(X, "N"), h.apply(X, "C")
    torch.cuda.synchronize()
    monkeypatch.setenv("BF_DISABLE_TMA", "1")
    Y2, Y2c = h.apply(X, "N"), h.apply(X, "C")
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2) and torch.equal(Y1c, Y2c)


@pytest.mark.parametrize("dtype", [np.complex128])
def test_fused_leaf_out_equals_separate(monkeypatch, dtype):
    """The row leaf fused into the last window pass and the separate leaf-out kernel compute the
    same products in the same order: bit-identical results (op N and C, permuted rows)."""
    bf = random_butterfly(L=6, leaf=32, r=16, seed=5, dtype=dtype)
    bf.row_perm = np.random.default_rng(1).permutation(bf.m).astype(np.int64)
    X = dev(random_rhs(bf.n, 40, seed=6, dtype=dtype))
    h1 = pkg.BFHandle(bf)
    Y1, Y1c = h1.apply(X, "N"), h1.apply(X, "C")
    torch.cuda.synchronize()
    monkeypatch.setenv("BF_NO_FUSE_OUT", "1")
    h2 = pkg.BFHandle(bf)
    assert h2.rounds("N")[-1]["name"].startswith("k_leaf")
    Y2, Y2c = h2.apply(X, "N"), h2.apply(X, "C")
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2) and torch.equal(Y1c, Y2c)


@pytest.mark.parametrize("L,leaf", [(6, 32), (5, 64), (7, 16)])
def test_fused_leaf_in_equals_separate(monkeypatch, L, leaf):
    """complex128, contiguous leaves: the column leaf fused into the first window pass (X rows by
    2-D TMA tiles in the ring pages) equals the separate leaf kernel bit for bit, op N / C / T."""
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=L + leaf)
    K = oracle.bf_dense(bf)
    monkeypatch.setenv("BF_FUSE_IN", "1")  # opt-in (measured slower on config 5)
    h1 = pkg.BFHandle(bf)
    assert h1.rounds("N")[0]["name"].startswith("k_bf_pass"), h1.rounds("N")
    monkeypatch.delenv("BF_FUSE_IN")
    h2 = pkg.BFHandle(bf)
    assert h2.rounds("N")[0]["name"].startswith("k_leaf")
    for op, nr in (("N", 32), ("C", 45), ("T", 7)):
        X = dev(random_rhs(bf.n, nr, seed=nr))
        Y1, Y2 = h1.apply(X, op), h2.apply(X, op)
        torch.cuda.synchronize()
        assert oracle.rel_err(host(Y1), oracle.apply_op(K, host(X), op)) <= 1e-12, op
        assert torch.equal(Y1, Y2), op


def test_pad_policy_keeps_large_low_rank_generic():
    """pad_pays (plan.cu): a large butterfly of ranks 1-2 would stream ~100x its entries once
    padded to rank 16, so it stays on the generic kernels (and is stored once, unpadded); a
    small one is padded onto the fused kernels.  Both against the level-by-level oracle."""
    from oracle.stagewise import bf_apply_stagewise
    for L, expect_fused in ((9, False), (4, True)):
        nb = 1 << L
        bf = random_ranks_butterfly(L, np.full(nb, 16), np.full(nb, 16), seed=L, rmin=1, rmax=2)
        h = pkg.BFHandle(bf)
        fused = h.rounds("N")[0]["name"].startswith("k_leaf")
        assert fused == expect_fused, (L, h.rounds("N")[0]["name"])
        if not fused:
            assert h.info["device_bytes"] < 4 * bf.nnz() * 16 + (64 << 20)
        for op in "NC":
            X = random_rhs(bf.n if op == "N" else bf.m, 9, seed=3)
            err = oracle.rel_err(host(h.apply(dev(X), op)), bf_apply_stagewise(bf, X, op))
            assert err <= 1e-12, (L, op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_fused_only_releases_the_pool(dtype):
    """BF_CREATE_FUSED_ONLY: the fused records alone serve every op (bit-identical applies), the
    generic factor pool is gone from the device (device_bytes drops by the factor bytes) and
    extraction / export refuse the handle."""
    import ctypes as C
    from paper_2007_00202_b200.bfapply import BFError
    bf = random_butterfly(L=6, leaf=32, r=16, seed=9, dtype=dtype)
    cs = 16 if dtype == np.complex128 else 8
    h0 = pkg.BFHandle(bf)
    h1 = pkg.BFHandle(bf, fused_only=True)
    assert h0.info["device_bytes"] - h1.info["device_bytes"] == bf.nnz() * cs
    for op, nr in (("N", 32), ("C", 5), ("T", 16)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=4, dtype=dtype)
        np.testing.assert_array_equal(host(h1.apply(dev(X), op)), host(h0.apply(dev(X), op)))
    with pytest.raises(BFError):
        h1.extract(np.arange(3), np.arange(4))
    # a ragged butterfly that stays on the generic kernels keeps its pool
    rng = np.random.default_rng(1)
    bfr = random_ranks_butterfly(4, rng.integers(1, 20, 16), rng.integers(1, 20, 16), seed=1, rmin=1, rmax=30,
                                 dtype=dtype)
    hr = pkg.BFHandle(bfr, fused_only=True)
    X = random_rhs(bfr.n, 3, seed=2, dtype=dtype)
    assert oracle.rel_err(host(hr.apply(dev(X))), oracle.bf_apply(bfr, X)) <= TOL[dtype]
    assert hr.extract(np.arange(2), np.arange(3)).shape == (2, 3)


@pytest.mark.parametrize("L,leaf,lc", [(8, 16, None), (9, 16, 3), (8, 32, 6), (6, 16, 2)])
@pytest.mark.parametrize("nrhs", [5, 16, 40])
def test_c64_pair_shared_split(monkeypatch, L, leaf, lc, nrhs):
    """complex64 4-level windows: a warp runs the two outputs of one input pair in one k-loop
    (PAIRW, fast.cu), splitting each slab fragment once.  Same MMAs in the same order per
    accumulator as one slot per k-loop (BF_NO_PAIRW), so the results are bit-identical; both
    agree with the oracle (ops N / C / T)."""
    dtype = np.complex64
    bf = random_butterfly(L=L, leaf=leaf, r=16, seed=11 + L, dtype=dtype, lc=lc)
    Xh = random_rhs(bf.n, nrhs, seed=5, dtype=dtype)
    Xc = random_rhs(bf.m, nrhs, seed=6, dtype=dtype)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    outs = {}
    for v in (0, 1):
        if v:
            monkeypatch.setenv("BF_NO_PAIRW", "1")
        outs[v] = (host(h.apply(dev(Xh), "N")), host(h.apply(dev(Xc), "C")), host(h.apply(dev(Xc), "T")))
    monkeypatch.delenv("BF_NO_PAIRW", raising=False)
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    Y, Yc, Yt = outs[0]
    assert oracle.rel_err(Y, oracle.apply_op(K, Xh, "N")) <= TOL[dtype]
    assert oracle.rel_err(Yc, oracle.apply_op(K, Xc, "C")) <= TOL[dtype]
    assert oracle.rel_err(Yt, oracle.apply_op(K, Xc, "T")) <= TOL[dtype]
