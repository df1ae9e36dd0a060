"""CPU oracle for the butterfly / HOD-BF multi-RHS apply.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
It shares no code with ``paper_2007_00202_b200`` (the CUDA path); both read factors
from ``bfinputs`` (pure storage, no apply arithmetic).

What it computes, in complex128 throughout:
  * Butterfly, Eq. (3.1): at the centre level lc every block is
        K(O_tau, S_nu) = Uhat_{tau,nu} B_{tau,nu} Vthat_{tau,nu}
    with the nested bases of Eq. (3.2):
        Uhat_{tau,nu} = U_tau                                        (l = L)
                      = diag(Uhat_{2tau,nu>>1}, Uhat_{2tau+1,nu>>1}) R_{tau,nu}   (l < L)
        Vthat_{tau,nu} = Vt_nu                                       (l = 0)
                       = W_{tau,nu} diag(Vthat_{tau>>1,2nu}, Vthat_{tau>>1,2nu+1}) (l > 0)
    (children of tau are 2tau, 2tau+1; parent of nu is nu>>1 -- P:291-295).
    The blocks at level lc tile K (complementary low-rank partition).
    User order: K_user[row_perm[i], col_perm[j]] = K[i, j].  Forward Y = K_user X,
    adjoint Y = K_user^H X, transpose Y = K_user^T X.
  * HOD-BF: A = blkdiag(D_t) at the leaves of T_H plus, for every pair of
    siblings tau1, tau2 on every level, A(T_tau1, T_tau2) = B_tau1 (a butterfly over
    the sibling subtrees).  Y = A X / A^H X.
  * Sampled rows / columns for sizes whose dense K does not fit (C2 step 5): the same
    Eq. (3.1)-(3.2) definitions restricted to selected rows (or columns).
Parity pins for every function are in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

C128 = np.complex128


# ----------------------------------------------------------------------------------
# rank-chain validation (mirrors the checks the C-ABI documents)
# ----------------------------------------------------------------------------------
def validate(bf):
    L, lc = bf.L, bf.lc
    assert 0 <= lc <= L, "need 0 <= lc <= L"
    nb = 1 << L
    rl, cl = bf.row_leaf_ptr, bf.col_leaf_ptr
    assert len(rl) == nb + 1 and len(cl) == nb + 1
    assert rl[0] == 0 and cl[0] == 0 and rl[-1] == bf.m and cl[-1] == bf.n
    assert np.all(np.diff(rl) >= 0) and np.all(np.diff(cl) >= 0)
    assert np.array_equal(np.sort(bf.row_perm), np.arange(bf.m))
    assert np.array_equal(np.sort(bf.col_perm), np.arange(bf.n))
    for tau in range(nb):
        assert bf.Ub(tau).shape[0] == rl[tau + 1] - rl[tau]
    for nu in range(nb):
        assert bf.Vtb(nu).shape[1] == cl[nu + 1] - cl[nu]

    def r(l, tau, nu):
        return bf.Ub(tau).shape[1] if l == L else bf.Rb(l, tau, nu).shape[1]

    def c(l, tau, nu):
        return bf.Vtb(nu).shape[0] if l == 0 else bf.Wb(l, tau, nu).shape[0]

    for l in range(lc, L):
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                assert bf.Rb(l, tau, nu).shape[0] == r(l + 1, 2 * tau, nu >> 1) + r(l + 1, 2 * tau + 1, nu >> 1)
    for l in range(1, lc + 1):
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                assert bf.Wb(l, tau, nu).shape[1] == c(l - 1, tau >> 1, 2 * nu) + c(l - 1, tau >> 1, 2 * nu + 1)
    for tau in range(1 << lc):
        for nu in range(1 << (L - lc)):
            assert bf.Bb(tau, nu).shape == (r(lc, tau, nu), c(lc, tau, nu))


# ----------------------------------------------------------------------------------
# Eq. (3.2) nested bases
# ----------------------------------------------------------------------------------
class _Bases:
    def __init__(self, bf):
        self.bf = bf
        self.Um = {}
        self.Vm = {}

    def Uhat(self, l, tau, nu):
        """Uhat_{tau,nu}: |O_tau| x r^l_{tau,nu} (Eq. 3.2 left)."""
        key = (l, tau, nu)
        if key not in self.Um:
            bf = self.bf
            if l == bf.L:
                assert nu == 0
                val = np.asarray(bf.Ub(tau), dtype=C128)
            else:
                top = self.Uhat(l + 1, 2 * tau, nu >> 1)
                bot = self.Uhat(l + 1, 2 * tau + 1, nu >> 1)
                val = sla.block_diag(top, bot) @ np.asarray(bf.Rb(l, tau, nu), dtype=C128)
            self.Um[key] = val
        return self.Um[key]

    def Vthat(self, l, tau, nu):
        """Vthat_{tau,nu}: c^l_{tau,nu} x |S_nu| (Eq. 3.2 right)."""
        key = (l, tau, nu)
        if key not in self.Vm:
            bf = self.bf
            if l == 0:
                assert tau == 0
                val = np.asarray(bf.Vtb(nu), dtype=C128)
            else:
                left = self.Vthat(l - 1, tau >> 1, 2 * nu)
                right = self.Vthat(l - 1, tau >> 1, 2 * nu + 1)
                val = np.asarray(bf.Wb(l, tau, nu), dtype=C128) @ sla.block_diag(left, right)
            self.Vm[key] = val
        return self.Vm[key]


def _O(bf, l, tau):
    w = 1 << (bf.L - l)
    return int(bf.row_leaf_ptr[tau * w]), int(bf.row_leaf_ptr[(tau + 1) * w])


def _S(bf, lev, nu):
    """Column range of T_S node nu at T_S level `lev`."""
    w = 1 << (bf.L - lev)
    return int(bf.col_leaf_ptr[nu * w]), int(bf.col_leaf_ptr[(nu + 1) * w])


def bf_dense_tree(bf) -> np.ndarray:
    """K in tree order, assembled block by block at level lc (Eq. 3.1)."""
    L, lc = bf.L, bf.lc
    K = np.zeros((bf.m, bf.n), dtype=C128)
    bases = _Bases(bf)
    for tau in range(1 << lc):
        r0, r1 = _O(bf, lc, tau)
        for nu in range(1 << (L - lc)):
            c0, c1 = _S(bf, L - lc, nu)
            K[r0:r1, c0:c1] = bases.Uhat(lc, tau, nu) @ np.asarray(bf.Bb(tau, nu), dtype=C128) @ bases.Vthat(lc, tau, nu)
    return K


def bf_dense(bf) -> np.ndarray:
    """K_user: K_user[row_perm[i], col_perm[j]] = K_tree[i, j]."""
    Kt = bf_dense_tree(bf)
    K = np.zeros_like(Kt)
    K[np.ix_(bf.row_perm, bf.col_perm)] = Kt
    return K


def apply_op(K: np.ndarray, X: np.ndarray, op: str) -> np.ndarray:
    X = np.asarray(X, dtype=C128)
    if op == "N":
        return K @ X
    if op == "C":
        return K.conj().T @ X
    if op == "T":
        return K.T @ X
    raise ValueError(op)


def bf_apply(bf, X, op: str = "N") -> np.ndarray:
    """Y = K_user X (op N), K_user^H X (op C) or K_user^T X (op T)."""
    return apply_op(bf_dense(bf), X, op)


# ----------------------------------------------------------------------------------
# sampled rows / columns (C2 step 5)
# ----------------------------------------------------------------------------------
def _ranks(bf):
    """r^l (row side, l = lc..L) and c^l (column side, l = 0..lc) per canonical index."""
    L, lc = bf.L, bf.lc
    r = {L: np.asarray(bf.U.cols)}
    for l in range(lc, L):
        r[l] = np.asarray(bf.R[l - lc].cols)
    c = {0: np.asarray(bf.Vt.rows)}
    for l in range(1, lc + 1):
        c[l] = np.asarray(bf.W[l - 1].rows)
    return r, c


def _row_chains(bf, tree_rows):
    """Row p of Uhat_{tau_c(p), nu} for every nu at level lc (Eq. 3.2 left, restricted
    to one row): Uhat_{tau,nu}[p] = Uhat_{child,nu>>1}[p] R_{tau,nu}[rows of that child], where
    child = 2tau or 2tau+1 is the one containing p.  Rows are processed in groups that share
    their level-l node tau; returns {tau_c: (row positions, [per nu: s x r^lc_{tau_c,nu}])}."""
    L, lc = bf.L, bf.lc
    r, _ = _ranks(bf)
    leaf = np.searchsorted(bf.row_leaf_ptr, tree_rows, side="right") - 1
    groups = {}
    for tau in np.unique(leaf):
        sel = np.nonzero(leaf == tau)[0]
        o0 = int(bf.row_leaf_ptr[tau])
        groups[int(tau)] = (sel, [np.asarray(bf.Ub(int(tau)), dtype=C128)[tree_rows[sel] - o0, :]])
    for l in range(L - 1, lc - 1, -1):
        nxt = {}
        for tau in sorted({t >> 1 for t in groups}):
            sels, vecs = [], []
            for ch in (0, 1):
                g = groups.get(2 * tau + ch)
                if g is None:
                    continue
                sel, v = g
                out = []
                for nu in range(1 << (L - l)):
                    Rb = np.asarray(bf.Rb(l, tau, nu), dtype=C128)
                    rt = int(r[l + 1][bf.idx(l + 1, 2 * tau, nu >> 1)])
                    part = Rb[:rt, :] if ch == 0 else Rb[rt:, :]
                    out.append(v[nu >> 1] @ part)
                sels.append(sel)
                vecs.append(out)
            sel = np.concatenate(sels)
            v = [np.vstack([vv[nu] for vv in vecs]) for nu in range(1 << (L - l))]
            nxt[tau] = (sel, v)
        groups = nxt
    return groups


def _col_descend(bf, groups):
    """Push row vectors u (one per centre block (tau_c, nu), s x c^lc) down the column-side
    recursion Eq. (3.2) right: u Vthat_{tau,nu} = [(u W_{tau,nu})[:, :c_left]
    Vthat_{tau>>1,2nu}, (u W_{tau,nu})[:, c_left:] Vthat_{tau>>1,2nu+1}], down to the leaves,
    where u Vthat_{0,nu} = u Vt_nu.  Returns (row positions, [per leaf nu: s x n_nu])."""
    L, lc = bf.L, bf.lc
    _, c = _ranks(bf)
    for l in range(lc, 0, -1):
        nxt = {}
        for tau in sorted({t >> 1 for t in groups}):
            sels, vecs = [], []
            for ch in (0, 1):
                g = groups.get(2 * tau + ch)
                if g is None:
                    continue
                sel, u = g
                t = 2 * tau + ch
                out = [None] * (1 << (L - l + 1))
                for nu in range(1 << (L - l)):
                    P = u[nu] @ np.asarray(bf.Wb(l, t, nu), dtype=C128)
                    cl = int(c[l - 1][bf.idx(l - 1, tau, 2 * nu)])
                    out[2 * nu], out[2 * nu + 1] = P[:, :cl], P[:, cl:]
                sels.append(sel)
                vecs.append(out)
            sel = np.concatenate(sels)
            u = [np.vstack([vv[nu] for vv in vecs]) for nu in range(1 << (L - l + 1))]
            nxt[tau] = (sel, u)
        groups = nxt
    sel, u = groups[0]
    return sel, [u[nu] @ np.asarray(bf.Vtb(nu), dtype=C128) for nu in range(1 << L)]


def bf_rows_apply(bf, user_rows, X) -> np.ndarray:
    """(K_user X)[user_rows, :] without forming K: rows of Eq. (3.1) blocks.

    Row p (tree position) of the centre block K(O_tau_c, S_nu) is Uhat_{tau_c,nu}[p] B_{tau_c,nu}
    Vthat_{tau_c,nu} (Eq. 3.1): the row of Uhat by Eq. (3.2) left restricted to that
    row (_row_chains), times B, then pushed as a row vector through Eq. (3.2) right down to the
    column leaves (_col_descend) -- the nested bases of P:302-317 evaluated from the row side,
    never forming any Vthat.  The K row segment over leaf S_nu0 then multiplies X(S_nu0)."""
    L, lc = bf.L, bf.lc
    assert len(np.unique(user_rows)) == len(user_rows), "sampled rows must be unique"
    X = np.asarray(X, dtype=C128)
    inv_row = np.empty(bf.m, dtype=np.int64)
    inv_row[bf.row_perm] = np.arange(bf.m)
    tree_rows = inv_row[np.asarray(user_rows, dtype=np.int64)]
    Xt = X[bf.col_perm, :]                     # X in column-tree order
    out = np.zeros((len(tree_rows), X.shape[1]), dtype=C128)
    if len(tree_rows) == 0:
        return out
    groups = _row_chains(bf, tree_rows)
    # centre: u_{tau_c,nu} = Uhat[p] B_{tau_c,nu}
    cen = {tau: (sel, [v[nu] @ np.asarray(bf.Bb(tau, nu), dtype=C128) for nu in range(1 << (L - lc))])
           for tau, (sel, v) in groups.items()}
    sel, seg = _col_descend(bf, cen)
    acc = np.zeros((len(sel), X.shape[1]), dtype=C128)
    for nu in range(1 << L):
        c0, c1 = int(bf.col_leaf_ptr[nu]), int(bf.col_leaf_ptr[nu + 1])
        acc += seg[nu] @ Xt[c0:c1, :]
    out[sel] = acc
    return out


def _col_chains(bf, tree_cols):
    """Column q of Vthat_{tau,nu_c(q)} for every tau at level lc (Eq. 3.2 right, P:312-316,
    restricted to one column): Vthat_{tau,nu}[:, q] = W_{tau,nu}[:, cols of the child holding q]
    Vthat_{tau>>1,child}[:, q].  Groups share their T_S node; returns
    {nu_c: (column positions, [per tau: c^lc_{tau,nu_c} x s])}."""
    L, lc = bf.L, bf.lc
    _, c = _ranks(bf)
    leaf = np.searchsorted(bf.col_leaf_ptr, tree_cols, side="right") - 1
    groups = {}
    for nu in np.unique(leaf):
        sel = np.nonzero(leaf == nu)[0]
        s0 = int(bf.col_leaf_ptr[nu])
        groups[int(nu)] = (sel, [np.asarray(bf.Vtb(int(nu)), dtype=C128)[:, tree_cols[sel] - s0]])
    for l in range(1, lc + 1):
        nxt = {}
        for nu in sorted({v >> 1 for v in groups}):
            sels, vecs = [], []
            for ch in (0, 1):
                g = groups.get(2 * nu + ch)
                if g is None:
                    continue
                sel, v = g
                out = []
                for tau in range(1 << l):
                    Wb = np.asarray(bf.Wb(l, tau, nu), dtype=C128)
                    cl = int(c[l - 1][bf.idx(l - 1, tau >> 1, 2 * nu)])
                    part = Wb[:, :cl] if ch == 0 else Wb[:, cl:]
                    out.append(part @ v[tau >> 1])
                sels.append(sel)
                vecs.append(out)
            sel = np.concatenate(sels)
            v = [np.hstack([vv[tau] for vv in vecs]) for tau in range(1 << l)]
            nxt[nu] = (sel, v)
        groups = nxt
    return groups


def _row_ascend(bf, groups):
    """Push column vectors w (one per centre block (tau, nu_c), r^lc x s) up the row-side
    recursion Eq. (3.2) left: Uhat_{tau,nu} w = [Uhat_{2tau,nu>>1} (R w)[:r_top];
    Uhat_{2tau+1,nu>>1} (R w)[r_top:]], up to the row leaves, where Uhat_{tau,0} = U_tau.
    Returns (column positions, [per leaf tau: m_tau x s])."""
    L, lc = bf.L, bf.lc
    r, _ = _ranks(bf)
    for l in range(lc, L):
        nxt = {}
        for nu in sorted({v >> 1 for v in groups}):
            sels, vecs = [], []
            for ch in (0, 1):
                g = groups.get(2 * nu + ch)
                if g is None:
                    continue
                sel, w = g
                v = 2 * nu + ch
                out = [None] * (1 << (l + 1))
                for tau in range(1 << l):
                    P = np.asarray(bf.Rb(l, tau, v), dtype=C128) @ w[tau]
                    rt = int(r[l + 1][bf.idx(l + 1, 2 * tau, nu)])
                    out[2 * tau], out[2 * tau + 1] = P[:rt], P[rt:]
                sels.append(sel)
                vecs.append(out)
            sel = np.concatenate(sels)
            w = [np.hstack([vv[tau] for vv in vecs]) for tau in range(1 << (l + 1))]
            nxt[nu] = (sel, w)
        groups = nxt
    sel, w = groups[0]
    return sel, [np.asarray(bf.Ub(tau), dtype=C128) @ w[tau] for tau in range(1 << L)]


def bf_cols_apply_adj(bf, user_cols, X) -> np.ndarray:
    """(K_user^H X)[user_cols, :] via sampled columns of Eq. (3.1) blocks: column q of the centre
    block K(O_tau, S_nu_c) is Uhat_{tau,nu_c} B_{tau,nu_c} Vthat_{tau,nu_c}[:, q] -- the column of
    Vthat by Eq. (3.2) right restricted to q (_col_chains), times B, pushed up Eq. (3.2) left to
    the row leaves (_row_ascend); then (K^H X)[q] = sum over row leaves K(O_tau, q)^H X(O_tau)."""
    L, lc = bf.L, bf.lc
    assert len(np.unique(user_cols)) == len(user_cols), "sampled columns must be unique"
    X = np.asarray(X, dtype=C128)
    inv_col = np.empty(bf.n, dtype=np.int64)
    inv_col[bf.col_perm] = np.arange(bf.n)
    tree_cols = inv_col[np.asarray(user_cols, dtype=np.int64)]
    Xt = X[bf.row_perm, :]                     # X in row-tree order
    out = np.zeros((len(tree_cols), X.shape[1]), dtype=C128)
    if len(tree_cols) == 0:
        return out
    groups = _col_chains(bf, tree_cols)
    cen = {nu: (sel, [np.asarray(bf.Bb(tau, nu), dtype=C128) @ v[tau] for tau in range(1 << lc)])
           for nu, (sel, v) in groups.items()}
    sel, seg = _row_ascend(bf, cen)
    acc = np.zeros((len(sel), X.shape[1]), dtype=C128)
    for tau in range(1 << L):
        r0, r1 = int(bf.row_leaf_ptr[tau]), int(bf.row_leaf_ptr[tau + 1])
        acc += seg[tau].conj().T @ Xt[r0:r1, :]
    out[sel] = acc
    return out


# ----------------------------------------------------------------------------------
# HOD-BF
# ----------------------------------------------------------------------------------
def hodbf_dense_tree(H) -> np.ndarray:
    """A in T_H tree order: blkdiag(D_t) + sibling off-diagonal butterflies."""
    A = np.zeros((H.n, H.n), dtype=C128)
    for t in range(1 << H.LH):
        a, b = int(H.leaf_ptr[t]), int(H.leaf_ptr[t + 1])
        A[a:b, a:b] = np.asarray(H.D.block(t), dtype=C128)
    for l in range(1, H.LH + 1):
        for tau in range(1 << l):
            r0, r1 = H.node_range(l, tau)
            c0, c1 = H.node_range(l, tau ^ 1)
            A[r0:r1, c0:c1] = bf_dense_tree(H.offdiag[l - 1][tau])
    return A


def hodbf_dense(H) -> np.ndarray:
    At = hodbf_dense_tree(H)
    A = np.zeros_like(At)
    A[np.ix_(H.perm, H.perm)] = At
    return A


def hodbf_apply(H, X, op: str = "N") -> np.ndarray:
    """Y = A X (op N) or A^H X (op C) or A^T X (op T), block by block.

    Never forms the full A: Y(T_t) = D_t X(T_t) at the leaves, and for every sibling
    pair Y(T_tau1) += B_tau1 X(T_tau2) (adjoint: Y(T_tau2) += B_tau1^H X(T_tau1)), with
    each B densified by Eq. (3.1)-(3.2).
    """
    X = np.asarray(X, dtype=C128)
    Xt = X[H.perm, :]
    Yt = np.zeros_like(Xt)
    for t in range(1 << H.LH):
        a, b = int(H.leaf_ptr[t]), int(H.leaf_ptr[t + 1])
        Yt[a:b] += apply_op(np.asarray(H.D.block(t), dtype=C128), Xt[a:b], op)
    for l in range(1, H.LH + 1):
        for tau in range(1 << l):
            r0, r1 = H.node_range(l, tau)
            c0, c1 = H.node_range(l, tau ^ 1)
            Kb = bf_dense_tree(H.offdiag[l - 1][tau])
            if op == "N":
                Yt[r0:r1] += Kb @ Xt[c0:c1]
            elif op == "C":
                Yt[c0:c1] += Kb.conj().T @ Xt[r0:r1]
            else:
                Yt[c0:c1] += Kb.T @ Xt[r0:r1]
    Y = np.zeros_like(Yt)
    Y[H.perm, :] = Yt
    return Y


def hodbf_rows_apply(H, user_rows, X) -> np.ndarray:
    """(A X)[user_rows, :] for an HOD-BF too large to densify (config 4):
    row p of A (tree order) = row p of its leaf block D_t, plus, at every level l, row p of
    the sibling butterfly A(T_tau, T_{tau^1}) of the node tau containing p, each
    evaluated with bf_rows_apply on that butterfly (tree-local, identity perms)."""
    X = np.asarray(X, dtype=C128)
    user_rows = np.asarray(user_rows, dtype=np.int64)
    assert len(np.unique(user_rows)) == len(user_rows), "sampled rows must be unique"
    inv = np.empty(H.n, dtype=np.int64)
    inv[H.perm] = np.arange(H.n)
    tree = inv[user_rows]
    Xt = X[H.perm, :]
    out = np.zeros((len(tree), X.shape[1]), dtype=C128)
    leaf = np.searchsorted(H.leaf_ptr, tree, side="right") - 1
    for t in np.unique(leaf):
        sel = np.nonzero(leaf == t)[0]
        a, b = int(H.leaf_ptr[t]), int(H.leaf_ptr[t + 1])
        out[sel] += np.asarray(H.D.block(int(t)), dtype=C128)[tree[sel] - a, :] @ Xt[a:b]
    for l in range(1, H.LH + 1):
        node = leaf >> (H.LH - l)
        for tau in np.unique(node):
            sel = np.nonzero(node == tau)[0]
            r0, r1 = H.node_range(l, int(tau))
            c0, c1 = H.node_range(l, int(tau) ^ 1)
            out[sel] += bf_rows_apply(H.offdiag[l - 1][int(tau)], tree[sel] - r0, Xt[c0:c1])
    return out


def rel_err(Y, Yref) -> float:
    """||Y - Yref||_F / ||Yref||_F (the parity metric)."""
    Yref = np.asarray(Yref, dtype=C128)
    nrm = np.linalg.norm(Yref)
    return float(np.linalg.norm(np.asarray(Y, dtype=C128) - Yref) / (nrm if nrm > 0 else 1.0))


def bf_extract(bf, user_rows, user_cols) -> np.ndarray:
    """K_user(user_rows, user_cols): the sub-matrix extract_BF returns (Alg. 3, P:472-526;
    SURVEY 8(f) NEXT-1), by its plain definition -- the entries of K (Eq. 3.1-3.2) at the requested
    rows and columns.  Rows of K through bf_rows_apply (Eq. 3.2 restricted to those rows) times
    unit columns; repeated indices allowed."""
    rows = np.asarray(user_rows, dtype=np.int64)
    cols = np.asarray(user_cols, dtype=np.int64)
    ur, inv = np.unique(rows, return_inverse=True)
    E = np.zeros((bf.n, len(cols)), dtype=C128)
    E[cols, np.arange(len(cols))] = 1.0
    return bf_rows_apply(bf, ur, E)[inv]


def hodbf_extract(H, user_rows, user_cols) -> np.ndarray:
    """A(user_rows, user_cols) of an HOD-BF (extract_HODBF) by its
    plain definition: the entries of the assembled matrix."""
    A = hodbf_dense(H)
    return A[np.ix_(np.asarray(user_rows, dtype=np.int64), np.asarray(user_cols, dtype=np.int64))]

