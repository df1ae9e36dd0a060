"""CPU level-by-level butterfly / HOD-BF apply: the secondary full-vector oracle.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.  It shares
no code with ``oracle/dense.py`` (nor with the CUDA path): both read the factor containers of
``bfinputs`` (storage only) and nothing else.

What it computes: the O(n log n) apply of P:354 ("the storage and
application costs of a matrix-vector product scale as O(n log n)"), i.e. the product of the
factors of Eq. (3.3)

    K = U^L R^{L-1} ... R^{lc} B^{lc} W^{lc} ... W^1 V^0

applied stage by stage to a block of right-hand sides, in complex128, with the stage
recursions of Eq. (3.2) written blockwise:

  a1  z^0_{0,nu}      = Vt_nu X(S_nu)                                   (V^0)
  a2  z^l_{tau,nu}    = W_{tau,nu} [z^{l-1}_{tau>>1,2nu}; z^{l-1}_{tau>>1,2nu+1}]   l = 1..lc
                                                                       (W^l)
  a3  y^{lc}_{tau,nu} = B_{tau,nu} z^{lc}_{tau,nu}                      (B^{lc})
  a4  [y^{l+1}_{2tau,nu>>1}; y^{l+1}_{2tau+1,nu>>1}] += R_{tau,nu} y^l_{tau,nu}   l = lc..L-1
                                                                       (R^l)
  a5  Y(O_tau)        = U_tau y^L_{tau,0}                               (U^L)

and the conjugate transpose (a6) as the same stages in reverse order with every factor
conjugate-transposed; op T = conj(op C (conj X)).  User order: X is read through col_perm,
Y written through row_perm (K_user[row_perm[i], col_perm[j]] = K_tree[i, j]).

Blocks are addressed canonically (level l, idx = tau * 2^(L-l) + nu; SURVEY 8(a) notation).
When every block of a stage has the same shape (configs 1 and 5) the stage is one batched
matmul over the stacked blocks (same arithmetic, the independent block products split across
host threads); otherwise it is a loop over blocks.  Both forms are pinned against
``oracle.dense.bf_dense`` in tests/test_oracle_stagewise.py.

HOD-BF: Y = blkdiag(D) X + sum over levels and sibling pairs of the
off-diagonal butterflies applied by the same stage recursion.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

C128 = np.complex128


def host_threads() -> int:
    """Threads the batched stages use: the cores this process may run on."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


# ----------------------------------------------------------------------------------
# block access (canonical order, column-major packed stages of bfinputs.Stage)
# ----------------------------------------------------------------------------------
def _blk(stage, i):
    r, c, o = int(stage.rows[i]), int(stage.cols[i]), int(stage.offs[i])
    return np.asarray(stage.data[o:o + r * c], dtype=C128).reshape(c, r).T


def _stack(stage):
    """All blocks of a uniform stage as an (nblocks, rows, cols) array, else None."""
    if stage.nblocks == 0 or np.any(stage.rows != stage.rows[0]) or np.any(stage.cols != stage.cols[0]):
        return None
    r, c = int(stage.rows[0]), int(stage.cols[0])
    return np.asarray(stage.data, dtype=C128).reshape(stage.nblocks, c, r).transpose(0, 2, 1)


class _Pool:
    """Batched block products A[b] @ Z[b] split into chunks over host threads."""

    def __init__(self, threads):
        self.threads = threads or host_threads()
        self.ex = ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    def bmm(self, A, Z):
        out = np.empty(A.shape[:-1] + Z.shape[-1:], dtype=C128)
        n = A.shape[0]
        if self.ex is None or n < 2 * self.threads:
            np.matmul(A, Z, out=out)
            return out
        step = (n + self.threads - 1) // self.threads
        futs = [self.ex.submit(np.matmul, A[s:s + step], Z[s:s + step], out=out[s:s + step])
                for s in range(0, n, step)]
        for f in futs:
            f.result()
        return out

    def close(self):
        if self.ex is not None:
            self.ex.shutdown()


def _uniform(bf):
    """True when every stage is uniform and the leaves are of one size (batched form)."""
    st = [bf.U, bf.B, bf.Vt] + list(bf.R) + list(bf.W)
    if any(_stack_shape(s) is None for s in st):
        return False
    return len(np.unique(np.diff(bf.row_leaf_ptr))) == 1 and len(np.unique(np.diff(bf.col_leaf_ptr))) == 1


def _stack_shape(stage):
    if stage.nblocks == 0 or np.any(stage.rows != stage.rows[0]) or np.any(stage.cols != stage.cols[0]):
        return None
    return int(stage.rows[0]), int(stage.cols[0])


# ----------------------------------------------------------------------------------
# forward apply, per block (any ranks, any leaves)
# ----------------------------------------------------------------------------------
def _fwd_blocks(bf, Xt):
    L, lc = bf.L, bf.lc
    nb = 1 << L
    k = Xt.shape[1]
    cl, rl = bf.col_leaf_ptr, bf.row_leaf_ptr
    # a1: level 0 (tau = 0, nu = 0..2^L-1)
    z = [_blk(bf.Vt, nu) @ Xt[int(cl[nu]):int(cl[nu + 1])] for nu in range(nb)]
    # a2: W stages
    for l in range(1, lc + 1):
        W = bf.W[l - 1]
        wp, wc = 1 << (L - l + 1), 1 << (L - l)   # nu count at level l-1 and at level l
        zn = [None] * nb
        for tau in range(1 << l):
            for nu in range(wc):
                i = tau * wc + nu
                p = (tau >> 1) * wp
                zn[i] = _blk(W, i) @ np.vstack([z[p + 2 * nu], z[p + 2 * nu + 1]])
        z = zn
    # a3: centre
    y = [_blk(bf.B, i) @ z[i] for i in range(nb)]
    # a4: R stages, scatter-add into the two children of tau
    for l in range(lc, L):
        R = bf.R[l - lc]
        wc, wn = 1 << (L - l), 1 << (L - l - 1)  # nu count at level l and at level l+1
        yn = [None] * nb
        for tau in range(1 << l):
            for nu in range(wc):
                i = tau * wc + nu
                P = _blk(R, i) @ y[i]
                top = (2 * tau) * wn + (nu >> 1)
                bot = (2 * tau + 1) * wn + (nu >> 1)
                rt = _rank_row(bf, l + 1, top)
                for j, part in ((top, P[:rt]), (bot, P[rt:])):
                    yn[j] = part.copy() if yn[j] is None else yn[j] + part
        y = yn
    # a5: row leaves
    Yt = np.zeros((bf.m, k), dtype=C128)
    for tau in range(nb):
        Yt[int(rl[tau]):int(rl[tau + 1])] = _blk(bf.U, tau) @ y[tau]
    return Yt


def _rank_row(bf, l, i):
    """r^l at canonical index i: columns of U_tau (l = L) or of R_{tau,nu} (l < L)."""
    return int(bf.U.cols[i]) if l == bf.L else int(bf.R[l - bf.lc].cols[i])


def _rank_col(bf, l, i):
    """c^l at canonical index i: rows of Vt_nu (l = 0) or of W_{tau,nu} (l > 0)."""
    return int(bf.Vt.rows[i]) if l == 0 else int(bf.W[l - 1].rows[i])


# ----------------------------------------------------------------------------------
# adjoint apply, per block: the stages of _fwd_blocks reversed, factors conjugate-transposed
# ----------------------------------------------------------------------------------
def _adj_blocks(bf, Xt):
    L, lc = bf.L, bf.lc
    nb = 1 << L
    k = Xt.shape[1]
    cl, rl = bf.col_leaf_ptr, bf.row_leaf_ptr
    # a5^H: y^L_tau = U_tau^H X(O_tau)
    y = [_blk(bf.U, tau).conj().T @ Xt[int(rl[tau]):int(rl[tau + 1])] for tau in range(nb)]
    # a4^H: y^l_{tau,nu} = R_{tau,nu}^H [y^{l+1}_{2tau,nu>>1}; y^{l+1}_{2tau+1,nu>>1}], l = L-1..lc
    for l in range(L - 1, lc - 1, -1):
        R = bf.R[l - lc]
        wc, wn = 1 << (L - l), 1 << (L - l - 1)
        yn = [None] * nb
        for tau in range(1 << l):
            for nu in range(wc):
                i = tau * wc + nu
                top = (2 * tau) * wn + (nu >> 1)
                bot = (2 * tau + 1) * wn + (nu >> 1)
                yn[i] = _blk(R, i).conj().T @ np.vstack([y[top], y[bot]])
        y = yn
    # a3^H
    z = [_blk(bf.B, i).conj().T @ y[i] for i in range(nb)]
    # a2^H: [z^{l-1}_{tau>>1,2nu}; z^{l-1}_{tau>>1,2nu+1}] += W_{tau,nu}^H z^l_{tau,nu}, l = lc..1
    for l in range(lc, 0, -1):
        W = bf.W[l - 1]
        wp, wc = 1 << (L - l + 1), 1 << (L - l)
        zn = [None] * nb
        for tau in range(1 << l):
            for nu in range(wc):
                i = tau * wc + nu
                P = _blk(W, i).conj().T @ z[i]
                p = (tau >> 1) * wp
                left, right = p + 2 * nu, p + 2 * nu + 1
                cL = _rank_col(bf, l - 1, left)
                for j, part in ((left, P[:cL]), (right, P[cL:])):
                    zn[j] = part.copy() if zn[j] is None else zn[j] + part
        z = zn
    # a1^H: Y(S_nu) = Vt_nu^H z^0_nu
    Yt = np.zeros((bf.n, k), dtype=C128)
    for nu in range(nb):
        Yt[int(cl[nu]):int(cl[nu + 1])] = _blk(bf.Vt, nu).conj().T @ z[nu]
    return Yt


# ----------------------------------------------------------------------------------
# batched forms (uniform stages): slabs of level l as an array (2^l, 2^(L-l), rank, k)
# ----------------------------------------------------------------------------------
def _fwd_batched(bf, Xt, pool):
    L, lc = bf.L, bf.lc
    nb = 1 << L
    k = Xt.shape[1]
    leaf_c = int(bf.col_leaf_ptr[1])
    leaf_r = int(bf.row_leaf_ptr[1])
    # a1
    Z = pool.bmm(_stack(bf.Vt), Xt.reshape(nb, leaf_c, k))           # (nb, c0, k), idx = nu
    for l in range(1, lc + 1):
        Wst = _stack(bf.W[l - 1])                                       # (nb, c, 2c') idx = tau 2^(L-l) + nu
        c_in = Z.shape[1]
        # input pair of (tau, nu) = level l-1 slabs (tau>>1, 2nu), (tau>>1, 2nu+1), stacked rows
        Zp = Z.reshape(1 << (l - 1), 1 << (L - l), 2 * c_in, k)      # (tau>>1, nu, 2c', k)
        Zin = np.repeat(Zp[:, None], 2, axis=1).reshape(nb, 2 * c_in, k)  # tau = 2 (tau>>1) + s
        Z = pool.bmm(Wst, Zin)
    # a3
    Y = pool.bmm(_stack(bf.B), Z)
    for l in range(lc, L):
        Rst = _stack(bf.R[l - lc])                                      # (nb, 2r', r)
        P = pool.bmm(Rst, Y)                                            # (nb, 2r', k) idx = tau 2^(L-l) + nu
        r_out = P.shape[1] // 2
        # P[tau, nu', s, child, r', k] with nu = 2nu' + s; out (2tau + child, nu') = sum_s
        P = P.reshape(1 << l, 1 << (L - l - 1), 2, 2, r_out, k).sum(axis=2)
        Y = np.ascontiguousarray(P.transpose(0, 2, 1, 3, 4)).reshape(nb, r_out, k)
    # a5
    return pool.bmm(_stack(bf.U), Y).reshape(nb * leaf_r, k)


def _adj_batched(bf, Xt, pool):
    L, lc = bf.L, bf.lc
    nb = 1 << L
    k = Xt.shape[1]
    leaf_c = int(bf.col_leaf_ptr[1])
    leaf_r = int(bf.row_leaf_ptr[1])
    H = lambda A: np.conj(A).transpose(0, 2, 1)  # noqa: E731  (blockwise conjugate transpose)
    Y = pool.bmm(H(_stack(bf.U)), Xt.reshape(nb, leaf_r, k))         # (nb, rL, k), idx = tau
    for l in range(L - 1, lc - 1, -1):
        Rst = _stack(bf.R[l - lc])
        r_in = Y.shape[1]
        # level l+1 slabs (tau', nu'): input of (tau, nu) = [(2tau, nu>>1); (2tau+1, nu>>1)]
        Yp = Y.reshape(1 << l, 2, 1 << (L - l - 1), r_in, k).transpose(0, 2, 1, 3, 4)
        Yp = Yp.reshape(1 << l, 1 << (L - l - 1), 2 * r_in, k)
        Yin = np.repeat(Yp[:, :, None], 2, axis=2).reshape(nb, 2 * r_in, k)  # nu = 2 (nu>>1) + s
        Y = pool.bmm(H(Rst), Yin)
    Z = pool.bmm(H(_stack(bf.B)), Y)
    for l in range(lc, 0, -1):
        Wst = _stack(bf.W[l - 1])
        P = pool.bmm(H(Wst), Z)                                         # (nb, 2c', k) idx = tau 2^(L-l) + nu
        c_out = P.shape[1] // 2
        # out (tau>>1, 2nu + half) = sum over tau's two values 2(tau>>1) + s
        P = P.reshape(1 << (l - 1), 2, 1 << (L - l), 2, c_out, k).sum(axis=1)
        Z = P.reshape(nb, c_out, k)
    return pool.bmm(H(_stack(bf.Vt)), Z).reshape(nb * leaf_c, k)


# ----------------------------------------------------------------------------------
# public entry points
# ----------------------------------------------------------------------------------
def bf_apply_stagewise(bf, X, op: str = "N", threads=None, batched=None) -> np.ndarray:
    """Y = K_user X (op N), K_user^H X (op C) or K_user^T X (op T), stage by stage.

    ``batched``: None picks the batched form when every stage is uniform; False forces the
    per-block loops (the pins exercise both)."""
    X = np.asarray(X, dtype=C128)
    if op == "T":
        return np.conj(bf_apply_stagewise(bf, np.conj(X), "C", threads, batched))
    if op not in ("N", "C"):
        raise ValueError(op)
    use_b = _uniform(bf) if batched is None else (batched and _uniform(bf))
    if op == "N":
        Xt = np.ascontiguousarray(X[bf.col_perm, :])
    else:
        Xt = np.ascontiguousarray(X[bf.row_perm, :])
    if use_b:
        pool = _Pool(threads)
        try:
            Yt = (_fwd_batched if op == "N" else _adj_batched)(bf, Xt, pool)
        finally:
            pool.close()
    else:
        Yt = (_fwd_blocks if op == "N" else _adj_blocks)(bf, Xt)
    Y = np.empty_like(Yt)
    Y[bf.row_perm if op == "N" else bf.col_perm, :] = Yt
    return Y


def hodbf_apply_stagewise(H, X, op: str = "N", threads=None) -> np.ndarray:
    """Y = A X / A^H X / A^T X for the HOD-BF matrix of P:542 without densifying anything:
    the dense leaf diagonals D_t times X(T_t), plus every sibling pair's off-diagonal
    butterflies applied stage by stage (op N: Y(T_tau) += B_tau X(T_{tau^1}); op C:
    Y(T_{tau^1}) += B_tau^H X(T_tau))."""
    X = np.asarray(X, dtype=C128)
    if op == "T":
        return np.conj(hodbf_apply_stagewise(H, np.conj(X), "C", threads))
    Xt = X[H.perm, :]
    Yt = np.zeros_like(Xt)
    for t in range(1 << H.LH):
        a, b = int(H.leaf_ptr[t]), int(H.leaf_ptr[t + 1])
        D = _blk(H.D, t)
        Yt[a:b] += (D if op == "N" else D.conj().T) @ Xt[a:b]
    for l in range(1, H.LH + 1):
        w = 1 << (H.LH - l)
        for tau in range(1 << l):
            r0, r1 = int(H.leaf_ptr[tau * w]), int(H.leaf_ptr[(tau + 1) * w])
            s = tau ^ 1
            c0, c1 = int(H.leaf_ptr[s * w]), int(H.leaf_ptr[(s + 1) * w])
            Bt = H.offdiag[l - 1][tau]
            # off-diagonal butterflies are tree-local: identity perms (bfinputs.HODBF)
            assert np.array_equal(Bt.row_perm, np.arange(Bt.m)) and np.array_equal(Bt.col_perm, np.arange(Bt.n))
            if op == "N":
                Yt[r0:r1] += bf_apply_stagewise(Bt, Xt[c0:c1], "N", threads)
            else:
                Yt[c0:c1] += bf_apply_stagewise(Bt, Xt[r0:r1], "C", threads)
    Y = np.empty_like(Yt)
    Y[H.perm, :] = Yt
    return Y
