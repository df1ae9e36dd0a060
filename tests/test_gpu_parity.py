"""GPU parity: libbfapply (through the C-ABI) vs the CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): relative Frobenius error <= 1e-12 for complex128 and
<= 1e-5 for complex64.  For c64 the oracle runs in c128 on the c64-rounded factors and
inputs.  Closed-form pins (identity, DFT) are compared exactly / against
numpy.fft.  Full-size configs are compared on sampled rows / columns
and by the dot-product identity.
"""
import numpy as np
import pytest
import torch

import oracle
from bfinputs import (dft_butterfly, identity_butterfly, random_butterfly, random_ranks_butterfly,
                      random_rhs, butterfly_from_blocks)
from bfinputs.configs import cfg1, cfg2, cfg3, cfg4, cfg5, helmholtz_plane_hodbf
import paper_2007_00202_b200 as pkg

pytestmark = pytest.mark.gpu

TOL = {np.complex128: 1e-12, np.complex64: 1e-5}


def dev(X):
    """(rows, nrhs) numpy column-major block -> (nrhs, rows) contiguous CUDA tensor."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X).T)).cuda()


def host(Y):
    return Y.cpu().numpy().T


def run(h, X, op="N"):
    Y = h.apply(dev(X), op)
    torch.cuda.synchronize()
    return host(Y)


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("op", ["N", "C", "T"])
def test_cfg1(dtype, op):
    bf, X = cfg1(dtype)
    if op != "N":
        X = random_rhs(bf.m, 16, seed=20, dtype=dtype)
    h = pkg.BFHandle(bf)
    assert h.info["launches_n"] == bf.L + 3
    err = oracle.rel_err(run(h, X, op), oracle.bf_apply(bf, X, op))
    assert err <= TOL[dtype], err


# ------------------------------------------------------------------ closed-form pins
@pytest.mark.parametrize("L,m0", [(5, 4), (3, 3), (6, 1), (1, 2), (0, 5)])
def test_identity_exact(L, m0):
    bf = identity_butterfly(L, m0)
    h = pkg.BFHandle(bf)
    X = random_rhs(bf.n, 7, seed=1)
    np.testing.assert_array_equal(run(h, X, "N"), X)
    np.testing.assert_array_equal(run(h, X, "C"), X)


@pytest.mark.parametrize("L", [3, 5])
def test_identity_exact_fast_shape(L):
    """A rank-16, leaf-16 identity has the fused path's shape, but selection factors take the
    generic path (4M product), so the apply stays exact (pin P1); random factors of the same
    shape take the fused kernels."""
    bf = identity_butterfly(L, 16)
    h = pkg.BFHandle(bf)
    assert all(r["name"].startswith("k_stage_tile") for r in h.rounds("N")), h.rounds("N")
    X = random_rhs(bf.n, 33, seed=2)
    np.testing.assert_array_equal(run(h, X, "N"), X)
    np.testing.assert_array_equal(run(h, X, "C"), X)
    hr = pkg.BFHandle(random_butterfly(L=L, leaf=16, r=16, seed=L))
    assert hr.rounds("N")[0]["name"].startswith("k_leaf")


@pytest.mark.parametrize("L", [4, 10, 15])
def test_dft_vs_numpy_fft(L):
    bf = dft_butterfly(L)
    h = pkg.BFHandle(bf)
    X = random_rhs(bf.n, 4, seed=L)
    assert oracle.rel_err(run(h, X, "N"), np.fft.fft(X, axis=0)) <= 1e-13
    assert oracle.rel_err(run(h, X, "C"), bf.n * np.fft.ifft(X, axis=0)) <= 1e-13


def test_dft_full_vector_L20():
    """P3 at config-5 scale (n = 2^20): the whole output vector is pinned."""
    bf = dft_butterfly(20)
    h = pkg.BFHandle(bf)
    X = random_rhs(bf.n, 2, seed=3)
    assert oracle.rel_err(run(h, X, "N"), np.fft.fft(X, axis=0)) <= 1e-12
    assert oracle.rel_err(run(h, X, "C"), bf.n * np.fft.ifft(X, axis=0)) <= 1e-12


def test_dft_c64():
    bf = dft_butterfly(12, np.complex64)
    h = pkg.BFHandle(bf)
    X = random_rhs(bf.n, 8, seed=3, dtype=np.complex64)
    assert oracle.rel_err(run(h, X, "N"), np.fft.fft(X.astype(np.complex128), axis=0)) <= 1e-5


# ------------------------------------------------------------------ ragged ranks, perms, edge cases
@pytest.mark.parametrize("L,lc,seed,rmin,rmax", [(4, 2, 0, 1, 6), (5, 1, 1, 0, 9), (3, 3, 2, 1, 40),
                                                 (6, 3, 3, 2, 20), (2, 0, 4, 1, 70), (7, 3, 5, 1, 12)])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_ragged(L, lc, seed, rmin, rmax, dtype):
    rng = np.random.default_rng(seed)
    nb = 1 << L
    rows = rng.integers(0, 40, nb)
    cols = rng.integers(1, 40, nb)
    bf = random_ranks_butterfly(L, rows, cols, seed=seed, rmin=rmin, rmax=rmax, lc=lc, dtype=dtype)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 37), ("C", 33), ("T", 5)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=seed + 9, dtype=dtype)
        err = oracle.rel_err(run(h, X, op), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


def test_L0_dense_block():
    rng = np.random.default_rng(0)
    Bm = rng.standard_normal((70, 50)) + 1j * rng.standard_normal((70, 50))
    bf = butterfly_from_blocks(0, 0, [0, 70], [0, 50], rng.permutation(70), rng.permutation(50),
                               [np.eye(70)], {}, [Bm], {}, [np.eye(50)])
    h = pkg.BFHandle(bf)
    X = random_rhs(50, 40, seed=2)
    assert oracle.rel_err(run(h, X), oracle.bf_apply(bf, X)) <= 1e-13


@pytest.mark.parametrize("nrhs", [1, 2, 31, 32, 33, 65, 130])
def test_nrhs_edges(nrhs):
    bf, _ = cfg1()
    h = pkg.BFHandle(bf)
    X = random_rhs(bf.n, nrhs, seed=nrhs)
    assert oracle.rel_err(run(h, X), oracle.bf_apply(bf, X)) <= 1e-12


def test_nrhs_zero_and_strides():
    bf, X = cfg1()
    h = pkg.BFHandle(bf)
    Y0 = h.apply(torch.zeros((0, bf.n), dtype=torch.complex128, device="cuda"))
    assert Y0.shape == (0, bf.m)
    # ld > rows on both sides
    Xp = torch.zeros((16, bf.n + 7), dtype=torch.complex128, device="cuda")
    Xp[:, :bf.n] = dev(X)
    Yp = torch.full((16, bf.m + 3), 7.0, dtype=torch.complex128, device="cuda")
    h.apply(Xp[:, :bf.n], out=Yp[:, :bf.m])
    torch.cuda.synchronize()
    assert oracle.rel_err(host(Yp[:, :bf.m]), oracle.bf_apply(bf, X)) <= 1e-12
    assert torch.all(Yp[:, bf.m:] == 7.0)


def test_errors_on_device():
    bf, X = cfg1()
    h = pkg.BFHandle(bf)
    Xd = dev(X)
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(pkg.BFError) as e:
        h.apply(Xd, work=small)
    assert e.value.code == -1
    with pytest.raises(pkg.BFError):
        h.apply(Xd, out=Xd)   # aliasing (m == n here)


def test_host_e2e_matches_device():
    bf, X = cfg1()
    h = pkg.BFHandle(bf)
    Xh = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory()
    Y = h.apply_host(Xh, "N")
    torch.cuda.synchronize()
    assert oracle.rel_err(Y.numpy().T, oracle.bf_apply(bf, X)) <= 1e-12
    Z = random_rhs(bf.m, 16, seed=4)
    Ya = h.apply_host(torch.from_numpy(np.ascontiguousarray(Z.T)).pin_memory(), "C")
    torch.cuda.synchronize()
    assert oracle.rel_err(Ya.numpy().T, oracle.bf_apply(bf, Z, "C")) <= 1e-12


def test_concurrent_streams():
    bf, X = cfg1()
    h = pkg.BFHandle(bf)
    ref = oracle.bf_apply(bf, X)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    w1 = torch.empty(h.workspace_size(16), dtype=torch.uint8, device="cuda")
    w2 = torch.empty(h.workspace_size(16), dtype=torch.uint8, device="cuda")
    Xd = dev(X)
    torch.cuda.synchronize()
    outs = []
    for _ in range(4):
        with torch.cuda.stream(s1):
            outs.append(h.apply(Xd, work=w1, stream=s1))
        with torch.cuda.stream(s2):
            outs.append(h.apply(Xd, work=w2, stream=s2))
    torch.cuda.synchronize()
    for Y in outs:
        assert oracle.rel_err(host(Y), ref) <= 1e-12


# ------------------------------------------------------------------ config 5 (full size, sampled)
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_cfg5_sampled(dtype):
    bf, X = cfg5(dtype)
    h = pkg.BFHandle(bf)
    Y = run(h, X, "N")
    rng = np.random.default_rng(0)
    # all rows of one centre node's two leaves plus scattered rows in the same centre node
    w = bf.m >> bf.lc
    tc = 37
    rows = np.unique(np.concatenate([np.arange(tc * w, tc * w + 128),
                                     rng.choice(np.arange(tc * w, (tc + 1) * w), 64, replace=False)]))
    ref = oracle.bf_rows_apply(bf, rows, X)
    assert oracle.rel_err(Y[rows], ref) <= TOL[dtype]
    Z = random_rhs(bf.m, 32, seed=12, dtype=dtype)
    Ya = run(h, Z, "C")
    wc = bf.n >> (bf.L - bf.lc)
    cols = np.arange(5 * wc, 5 * wc + 96)
    refc = oracle.bf_cols_apply_adj(bf, cols, Z)
    assert oracle.rel_err(Ya[cols], refc) <= TOL[dtype]
    # dot-product identity over the full vectors (P5)
    lhs = np.vdot(Z.astype(np.complex128), Y.astype(np.complex128))
    rhs = np.vdot(Ya.astype(np.complex128), X.astype(np.complex128))
    assert abs(lhs - rhs) <= TOL[dtype] * np.linalg.norm(Z) * np.linalg.norm(Y)


# ------------------------------------------------------------------ config 2 (kernel butterfly)
def test_cfg2():
    bf, X = cfg2()
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    assert oracle.rel_err(run(h, X, "N"), K @ X) <= 1e-12
    Z = random_rhs(bf.m, 64, seed=21)
    assert oracle.rel_err(run(h, Z, "C"), K.conj().T @ Z) <= 1e-12


# ------------------------------------------------------------------ HOD-BF
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_hodbf_small(dtype):
    H = helmholtz_plane_hodbf(32, 16, 10.0, 1e-4)
    H = H.astype(dtype)
    h = pkg.HODBFHandle(H)
    A = oracle.hodbf_dense(H)
    for op, nr in (("N", 40), ("C", 33), ("T", 3)):
        X = random_rhs(H.n, nr, seed=3, dtype=dtype)
        err = oracle.rel_err(run(h, X, op), oracle.apply_op(A, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_cfg3(dtype):
    H, X = cfg3(dtype)
    h = pkg.HODBFHandle(H)
    assert oracle.rel_err(run(h, X, "N"), oracle.hodbf_apply(H, X, "N")) <= TOL[dtype]
    Z = random_rhs(H.n, 64, seed=31, dtype=dtype)
    assert oracle.rel_err(run(h, Z, "C"), oracle.hodbf_apply(H, Z, "C")) <= TOL[dtype]


def test_cfg4():
    """Config 4 (Maxwell-type front, 51200 unknowns, dyadic kernel, nrhs 512; constructed with
    512 proxy rows / columns per ID): sampled rows of A X against the
    HOD-BF sampled-row oracle, and the adjoint through <A X, Z> = <X, A^H Z>
    over full vectors."""
    H, X = cfg4(proxy_cap=512)
    h = pkg.HODBFHandle(H)
    Y = run(h, X, "N")
    rng = np.random.default_rng(4)
    rows = np.unique(np.concatenate([np.arange(int(H.leaf_ptr[5]), int(H.leaf_ptr[6])),
                                     np.arange(int(H.leaf_ptr[700]), int(H.leaf_ptr[701])),
                                     rng.choice(H.n, 48, replace=False)]))
    assert oracle.rel_err(Y[rows], oracle.hodbf_rows_apply(H, rows, X)) <= 1e-12
    Z = random_rhs(H.n, 8, seed=41)
    Ya = run(h, Z, "C")
    lhs = np.vdot(Z, Y[:, :8])
    rhs = np.vdot(Ya, X[:, :8])
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Z) * np.linalg.norm(Y[:, :8])


@pytest.mark.parametrize("fast", [True, False])
def test_host_apply_pipelined(fast):
    """Back-to-back bf_apply_host calls (pipelined: call k+1's H2D overlaps call k's D2H) on
    distinct host buffers, alternating op N and C, are all correct after one synchronise."""
    bf = random_butterfly(L=6, leaf=32, r=16 if fast else 8, seed=12)
    h = pkg.BFHandle(bf)
    K = oracle.bf_dense(bf)
    ops = ["N", "C", "N", "N", "C", "T"]
    Xs = [random_rhs(bf.n, 33, seed=40 + i) for i in range(len(ops))]
    Xh = [torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory() for X in Xs]
    Yh = [torch.empty((33, bf.n), dtype=torch.complex128).pin_memory() for _ in ops]
    work = torch.empty(h.workspace_size_host(33), dtype=torch.uint8, device="cuda")
    for x, y, op in zip(Xh, Yh, ops):
        h.apply_host(x, op, out=y, work=work)
    torch.cuda.synchronize()
    for X, y, op in zip(Xs, Yh, ops):
        assert oracle.rel_err(y.numpy().T, oracle.apply_op(K, X, op)) <= 1e-12, op


@pytest.mark.parametrize("kind", ["generic", "fast", "hodbf"])
def test_cuda_graph_replay(kind):
    """An apply captured into a CUDA graph (BFHandle.graph) replays to the direct result,
    bit for bit, after the static input is refilled."""
    if kind == "hodbf":
        H = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4)
        h, n = pkg.HODBFHandle(H), H.n
    else:
        bf = random_butterfly(L=5, leaf=32, r=16 if kind == "fast" else 8, seed=3)
        h, n = pkg.BFHandle(bf), bf.n
    X1 = dev(random_rhs(n, 24, seed=1))
    X2 = dev(random_rhs(n, 24, seed=2))
    gr = h.graph(X1.clone(), "N")
    gr.X.copy_(X2)
    Yg = gr.replay().clone()
    Yd = h.apply(X2, "N")
    torch.cuda.synchronize()
    assert torch.equal(Yg, Yd)
