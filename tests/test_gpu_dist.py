"""GPU parity of the distributed apply's kernels (bf_dist_apply_pre / _post) against the
CPU oracle, on ONE device: the P rank-local handles run one after another in this process
and the all-to-all is replayed as device copies between their workspaces (the same
send / recv regions NCCL moves; no rank ever waits on another).  World size 1 runs the
real DistBFHandle.apply with its self exchange."""
import numpy as np
import pytest
import torch

import oracle
from bfinputs import random_butterfly, random_ranks_butterfly, random_rhs
from paper_2007_00202_b200.dist import DistBFHandle

pytestmark = pytest.mark.gpu

TOL = {np.complex128: 1e-12, np.complex64: 1e-5}


def _subtree_perm(n, leaf_ptr, L, p, seed):
    rng = np.random.default_rng(seed)
    perm = np.empty(n, dtype=np.int64)
    w = 1 << (L - p)
    for g in range(1 << p):
        a, b = int(leaf_ptr[g * w]), int(leaf_ptr[(g + 1) * w])
        perm[a:b] = a + rng.permutation(b - a)
    return perm


def emulate(bf, X, op, P):
    """Run the P-rank split apply on device 0; returns the full (rows_out, nrhs) result."""
    hs = [DistBFHandle(bf, g, P, 0) for g in range(P)]
    nrhs = X.shape[1]
    dt = torch.complex128 if X.dtype == np.complex128 else torch.complex64
    works, outs = [], []
    for h in hs:
        ri, ro, ui, uo = h.local_rows(op)
        Xl = torch.from_numpy(np.ascontiguousarray(X[ui:ui + ri].T)).cuda()
        wb = h.layout(op, nrhs)[0]
        w = torch.zeros(max(wb, 1), dtype=torch.uint8, device="cuda")
        from paper_2007_00202_b200.bfapply import lib, OPS
        import ctypes as C
        rc = lib().bf_dist_apply_pre(h.h, OPS[op], nrhs, C.c_void_p(Xl.data_ptr()), max(ri, 1),
                                     C.c_void_p(w.data_ptr()), w.numel(), None)
        assert rc == 0, lib().bf_last_error()
        works.append(w)
    cs = hs[0].cs
    lay = [h.layout(op, nrhs) for h in hs]
    # replay the all-to-all: rank g's send chunk for q -> rank q's recv chunk from g
    for g in range(P):
        _, so, _, sc, _ = lay[g]
        soff = so
        for q in range(P):
            _, _, ro, _, rcq = lay[q]
            roff = ro + sum(rcq[:g]) * cs
            n = sc[q] * cs
            assert n == rcq[g] * cs
            works[q][roff:roff + n].copy_(works[g][soff:soff + n])
            soff += n
    rows_out = bf.m if op == "N" else bf.n
    Y = np.zeros((rows_out, nrhs), dtype=X.dtype)
    for h, w in zip(hs, works):
        ri, ro, ui, uo = h.local_rows(op)
        Yl = torch.zeros((nrhs, max(ro, 1)), dtype=dt, device="cuda")
        from paper_2007_00202_b200.bfapply import lib, OPS
        import ctypes as C
        rc = lib().bf_dist_apply_post(h.h, OPS[op], nrhs, C.c_void_p(Yl.data_ptr()), max(ro, 1),
                                      C.c_void_p(w.data_ptr()), w.numel(), None)
        assert rc == 0, lib().bf_last_error()
        torch.cuda.synchronize()
        Y[uo:uo + ro] = Yl[:, :ro].cpu().numpy().T
    return Y


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("kind", ["uniform", "ragged"])
def test_dist_emulated(kind, P, dtype):
    if kind == "uniform":
        bf = random_butterfly(L=7, leaf=16, r=16, seed=P, dtype=dtype)
    else:
        rng = np.random.default_rng(P)
        bf = random_ranks_butterfly(7, rng.integers(0, 9, 128), rng.integers(1, 9, 128), seed=P, rmin=1,
                                    rmax=9, dtype=dtype)
    p = P.bit_length() - 1
    bf.row_perm = _subtree_perm(bf.m, bf.row_leaf_ptr, bf.L, p, 1)
    bf.col_perm = _subtree_perm(bf.n, bf.col_leaf_ptr, bf.L, p, 2)
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 33), ("C", 20), ("T", 5)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=P + nr, dtype=dtype)
        err = oracle.rel_err(emulate(bf, X, op, P), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, err)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("P,L", [(2, 8), (4, 10), (8, 9)])
def test_dist_fast_emulated(P, L, dtype):
    """Uniform rank-16 butterflies take the fused split (leaf + window-pass kernels, half-slab
    exchange format); identity perms, so the leaf kernels move X / Y with TMA tiles."""
    bf = random_butterfly(L=L, leaf=16, r=16, seed=L + P, dtype=dtype)
    assert DistBFHandle(bf, 0, P, 0).slab_format() == 1
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 32), ("C", 45), ("T", 7), ("N", 16), ("C", 12)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=P + nr, dtype=dtype)
        err = oracle.rel_err(emulate(bf, X, op, P), oracle.apply_op(K, X, op))
        assert err <= TOL[dtype], (op, nr, err)


@pytest.mark.parametrize("op", ["N", "C"])
def test_dist_world1_self_exchange(op):
    bf = random_butterfly(L=6, leaf=16, r=16, seed=9)
    h = DistBFHandle(bf, 0, 1, 0)
    X = random_rhs(bf.n, 40, seed=4)
    Y = h.apply(torch.from_numpy(np.ascontiguousarray(X.T)).cuda(), op)
    torch.cuda.synchronize()
    assert oracle.rel_err(Y.cpu().numpy().T, oracle.bf_apply(bf, X, op)) <= 1e-12


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_hodbf(world):
    """RHS-sharded HOD-BF (config 4's multi-GPU layout): the ranks' column blocks, applied one
    after another on one device, assemble the full result."""
    from bfinputs.configs import helmholtz_plane_hodbf
    from paper_2007_00202_b200.dist import ShardedHODBF
    H = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4, ncomp=2)
    X = random_rhs(H.n, 37, seed=world)
    Y = np.zeros_like(X)
    for r in range(world):
        s = ShardedHODBF(H, r, world, 0)
        c0, c1 = s.columns(X.shape[1])
        Yl = s.apply(torch.from_numpy(np.ascontiguousarray(X[:, c0:c1].T)).cuda())
        torch.cuda.synchronize()
        Y[:, c0:c1] = Yl.cpu().numpy().T
    assert oracle.rel_err(Y, oracle.hodbf_apply(H, X)) <= 1e-12


def emulate_p2p(bf, X, op, P):
    """The fused peer-memory exchange on one device: every rank's pre writes its centre slabs
    straight into the other ranks' recv regions (here plain device buffers), then every post."""
    import ctypes as C
    from paper_2007_00202_b200.bfapply import lib, OPS
    from paper_2007_00202_b200.dist import _lib
    hs = [DistBFHandle(bf, g, P, 0) for g in range(P)]
    nrhs = X.shape[1]
    dt = torch.complex128 if X.dtype == np.complex128 else torch.complex64
    lay = [h.layout(op, nrhs) for h in hs]
    works = [torch.zeros(max(l[0], 1), dtype=torch.uint8, device="cuda") for l in lay]
    peers = (C.c_void_p * P)(*[w.data_ptr() + l[2] for w, l in zip(works, lay)])
    for h, w in zip(hs, works):
        ri, ro, ui, uo = h.local_rows(op)
        Xl = torch.from_numpy(np.ascontiguousarray(X[ui:ui + ri].T)).cuda()
        rc = _lib().bf_dist_apply_pre_p2p(h.h, OPS[op], nrhs, C.c_void_p(Xl.data_ptr()), max(ri, 1),
                                          C.c_void_p(w.data_ptr()), w.numel(), peers, None)
        assert rc == 0, lib().bf_last_error()
    torch.cuda.synchronize()
    rows_out = bf.m if op == "N" else bf.n
    Y = np.zeros((rows_out, nrhs), dtype=X.dtype)
    for h, w in zip(hs, works):
        ri, ro, ui, uo = h.local_rows(op)
        Yl = torch.zeros((nrhs, max(ro, 1)), dtype=dt, device="cuda")
        rc = lib().bf_dist_apply_post(h.h, OPS[op], nrhs, C.c_void_p(Yl.data_ptr()), max(ro, 1),
                                      C.c_void_p(w.data_ptr()), w.numel(), None)
        assert rc == 0, lib().bf_last_error()
        torch.cuda.synchronize()
        Y[uo:uo + ro] = Yl[:, :ro].cpu().numpy().T
    return Y


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("P,L", [(2, 8), (4, 10), (8, 9)])
def test_dist_p2p_emulated(P, L, dtype):
    """Fused peer-memory exchange (bf_dist_apply_pre_p2p) == the oracle, and == the all-to-all
    version bit for bit (same kernels, only where the slabs are stored differs)."""
    bf = random_butterfly(L=L, leaf=16, r=16, seed=L + P + 1, dtype=dtype)
    K = oracle.bf_dense(bf)
    for op, nr in (("N", 32), ("C", 45), ("T", 7)):
        X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=P + nr + 1, dtype=dtype)
        Yp = emulate_p2p(bf, X, op, P)
        assert oracle.rel_err(Yp, oracle.apply_op(K, X, op)) <= TOL[dtype], op
        np.testing.assert_array_equal(Yp, emulate(bf, X, op, P))


def emulate_tree_hodbf(H, X, op, P):
    """The tree-partitioned HOD-BF (dist.TreeHODBF) on one device: every rank's local HOD-BF and
    column sides, the grouped exchange replayed as device copies into the sibling ranks' recv
    regions, then every rank's row sides accumulated into its rows.  X, Y in user order."""
    from paper_2007_00202_b200.dist import TreeHODBF
    ts = [TreeHODBF(H, g, P, 0) for g in range(P)]
    nrhs = X.shape[1]
    Xt = X[H.perm]  # HOD-BF tree order
    Ys = []
    for t in ts:
        lo, hi = t.rows()
        Xl = torch.from_numpy(np.ascontiguousarray(Xt[lo:hi].T)).cuda()
        Ys.append(t.local.apply(Xl, op))
        t.pre(Xl, op)
    torch.cuda.synchronize()
    bufs = [t.buffers(op, nrhs) for t in ts]
    for g in range(P):
        for li, (sv, _) in enumerate(bufs[g]):
            for peer, view in sv:
                dst = [v for src, v in bufs[peer][li][1] if src == g]
                assert len(dst) == 1 and dst[0].numel() == view.numel()
                dst[0].copy_(view)
    torch.cuda.synchronize()
    Yt = np.zeros_like(Xt)
    for t, Yl in zip(ts, Ys):
        t.post(Yl, op)
        torch.cuda.synchronize()
        lo, hi = t.rows()
        Yt[lo:hi] = Yl.cpu().numpy().T
    Y = np.empty_like(Yt)
    Y[H.perm] = Yt
    return Y


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_tree_hodbf_emulated(P, dtype):
    """HOD-BF distributed by tree node: the P ranks' results assemble A X and
    A^H X of the CPU oracle."""
    from bfinputs.configs import helmholtz_plane_hodbf
    H = helmholtz_plane_hodbf(32, 16, 10.0, 1e-4).astype(dtype)
    for op in ("N", "C"):
        X = random_rhs(H.n, 19, seed=P, dtype=dtype)
        err = oracle.rel_err(emulate_tree_hodbf(H, X, op, P), oracle.hodbf_apply(H, X, op))
        assert err <= TOL[dtype], (op, err)


# ---- library-owned NCCL communicator (bf_create_dist / bf_apply_dist) -----------------------
@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_library_nccl_world1(fast, dtype):
    """bf_apply_dist with a communicator the library created (bf_nccl_comm_init over one rank):
    pre, grouped ncclSend / ncclRecv to itself, post -- one C-ABI call per apply.  It must equal
    the pre / torch exchange / post path bit for bit, and the oracle within the bar.  (One GPU: a
    multi-rank NCCL communicator needs one device per rank.)"""
    from paper_2007_00202_b200.dist import NcclComm
    if fast:
        bf = random_butterfly(L=6, leaf=32, r=16, seed=3, dtype=dtype)
    else:
        rng = np.random.default_rng(2)
        bf = random_ranks_butterfly(5, rng.integers(1, 20, 32), rng.integers(1, 20, 32), seed=2, rmin=1, rmax=12,
                                    dtype=dtype)
    comm = NcclComm(0)
    try:
        h1 = DistBFHandle(bf, 0, 1, 0, comm=comm)
        h0 = DistBFHandle(bf, 0, 1, 0)
        K = oracle.bf_dense(bf)
        for op, nr in (("N", 32), ("C", 7)):
            X = random_rhs(bf.n if op == "N" else bf.m, nr, seed=4, dtype=dtype)
            Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
            Y1 = h1.apply(Xd, op)
            Y0 = h0.apply(Xd, op)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(Y1.cpu().numpy(), Y0.cpu().numpy())
            assert oracle.rel_err(Y1.cpu().numpy().T, oracle.apply_op(K, X, op)) <= TOL[dtype]
        h1.close()
    finally:
        comm.close()


def test_apply_dist_one_rank_without_comm():
    """bf_create_dist with a NULL communicator is legal for one rank: bf_apply_dist's exchange is
    then a device copy inside the workspace."""
    import ctypes as C
    from paper_2007_00202_b200.bfapply import _Keep, make_desc, lib, OPS
    from paper_2007_00202_b200.dist import _lib
    bf = random_butterfly(L=4, leaf=16, r=16, seed=5)
    keep = _Keep()
    d = make_desc(bf, keep)
    h = C.c_void_p()
    assert _lib().bf_create_dist(C.byref(d), 0, 1, None, 0, C.byref(h)) == 0
    ref = DistBFHandle(bf, 0, 1, 0)
    X = random_rhs(bf.n, 5, seed=6)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = torch.empty((5, bf.m), dtype=torch.complex128, device="cuda")
    wb = ref.layout("N", 5)[0]
    w = torch.empty(max(wb, 1), dtype=torch.uint8, device="cuda")
    rc = _lib().bf_apply_dist(h, OPS["N"], 5, C.c_void_p(Xd.data_ptr()), bf.n, C.c_void_p(Y.data_ptr()), bf.m,
                              C.c_void_p(w.data_ptr()), w.numel(), None)
    assert rc == 0, lib().bf_last_error()
    Y0 = ref.apply(Xd, "N")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Y.cpu().numpy(), Y0.cpu().numpy())
    lib().bf_destroy(h)
