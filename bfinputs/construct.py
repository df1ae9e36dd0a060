"""CPU construction tooling (TOOL, not the hot path): interpolative decomposition and
BF_entry_eval / HODBF_entry_eval, used to build the factor inputs of configs 2-4.

  * ID_eps: truncated column-pivoted QR.  Row ID of M: QR of M^T,
    M ~= U M(I,:),  U = P [I ; (R11^{-1} R12)^T].  Column ID: QR of M,
    M ~= M(:,J) V^T, V^T = [I, R11^{-1} R12] P^T.  Truncation keeps |R_kk| >= eps |R_11|
    (relative).
  * BF_entry_eval (Alg. 2): outer-to-inner row IDs from level L down to lc,
    column IDs from level 0 up to lc, skeleton block B at lc.  Proxies: the full
    S_nu / O_tau (brute force, exact; SURVEY C3 "configs 2-3"), optionally capped.
  * HODBF_entry_eval: dense leaves plus BF_entry_eval on every sibling
    off-diagonal block A(T_tau, T_{tau^1}) of T_H.

This produces *inputs* for the apply; it never applies a butterfly.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import scipy.linalg as sla

from .factors import Butterfly, HODBF, Stage, butterfly_from_blocks


def _pivoted_qr(M):
    Q, R, P = sla.qr(M, mode="economic", pivoting=True, check_finite=False)
    return R, P


def _rank(R, eps):
    d = np.abs(np.diag(R))
    if d.size == 0 or d[0] == 0.0:
        return 0
    return int(np.count_nonzero(d >= eps * d[0]))


def row_id(M: np.ndarray, eps: float):
    """M ~= U @ M[I, :].  Returns (U, I)."""
    m = M.shape[0]
    if m == 0 or M.shape[1] == 0:
        return np.zeros((m, 0), dtype=M.dtype), np.zeros(0, dtype=np.int64)
    R, P = _pivoted_qr(M.T)
    k = max(_rank(R, eps), 1)
    k = min(k, m)
    T = sla.solve_triangular(R[:k, :k], R[:k, k:], check_finite=False)
    U = np.zeros((m, k), dtype=M.dtype)
    U[P[:k], np.arange(k)] = 1.0
    U[P[k:], :] = T.T
    return U, P[:k].astype(np.int64)


def col_id(M: np.ndarray, eps: float):
    """M ~= M[:, J] @ Vt.  Returns (Vt, J)."""
    n = M.shape[1]
    if n == 0 or M.shape[0] == 0:
        return np.zeros((0, n), dtype=M.dtype), np.zeros(0, dtype=np.int64)
    R, P = _pivoted_qr(M)
    k = max(_rank(R, eps), 1)
    k = min(k, n)
    T = sla.solve_triangular(R[:k, :k], R[:k, k:], check_finite=False)
    Vt = np.zeros((k, n), dtype=M.dtype)
    Vt[np.arange(k), P[:k]] = 1.0
    Vt[:, P[k:]] = T
    return Vt, P[:k].astype(np.int64)


def _proxy(idx: np.ndarray, cap: Optional[int], rng) -> np.ndarray:
    if cap is None or idx.size <= cap:
        return idx
    return np.sort(rng.choice(idx, size=cap, replace=False))


def bf_entry_eval(extract: Callable, row_leaf_ptr, col_leaf_ptr, L: int, eps: float,
                  lc: Optional[int] = None, proxy_cap: Optional[int] = None, seed: int = 0,
                  dtype=np.complex128, meta=None) -> Butterfly:
    """Alg. 2 BF_entry_eval on a matrix given by extract(I, J).

    I, J are tree positions (0..m-1, 0..n-1); the returned butterfly has identity
    perms (tree order == user order for its caller).  Skeletons are per block
    (SURVEY A6): O-bar_{tau,nu} and S-bar_{tau,nu}.
    """
    lc = L // 2 if lc is None else lc
    rng = np.random.default_rng(seed)
    rlp = np.asarray(row_leaf_ptr, dtype=np.int64)
    clp = np.asarray(col_leaf_ptr, dtype=np.int64)
    m, n = int(rlp[-1]), int(clp[-1])

    def O(l, tau):  # rows of T_O node tau at level l
        w = 1 << (L - l)
        return np.arange(rlp[tau * w], rlp[(tau + 1) * w])

    def S(l, nu):  # columns of T_S node nu at level l
        w = 1 << (L - l)
        return np.arange(clp[nu * w], clp[(nu + 1) * w])

    # ---- row side, l = L .. lc (left column of Alg. 2) ----
    Obar = {}
    U_blocks = []
    allS = np.arange(n)
    for tau in range(1 << L):
        rows = O(L, tau)
        cols = _proxy(allS, proxy_cap, rng)
        Ub, I = row_id(extract(rows, cols), eps)
        U_blocks.append(Ub)
        Obar[(L, tau, 0)] = rows[I]
    R_blocks = {}
    for l in range(L - 1, lc - 1, -1):
        blocks = []
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                rows = np.concatenate([Obar[(l + 1, 2 * tau, nu >> 1)], Obar[(l + 1, 2 * tau + 1, nu >> 1)]])
                cols = _proxy(S(L - l, nu), proxy_cap, rng)
                Rb, I = row_id(extract(rows, cols), eps)
                blocks.append(Rb)
                Obar[(l, tau, nu)] = rows[I]
        R_blocks[l] = blocks
    # ---- column side, l = 0 .. lc (right column of Alg. 2) ----
    Sbar = {}
    Vt_blocks = []
    allO = np.arange(m)
    for nu in range(1 << L):
        cols = S(L, nu)
        rows = _proxy(allO, proxy_cap, rng)
        Vb, J = col_id(extract(rows, cols), eps)
        Vt_blocks.append(Vb)
        Sbar[(0, 0, nu)] = cols[J]
    W_blocks = {}
    for l in range(1, lc + 1):
        blocks = []
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                cols = np.concatenate([Sbar[(l - 1, tau >> 1, 2 * nu)], Sbar[(l - 1, tau >> 1, 2 * nu + 1)]])
                rows = _proxy(O(l, tau), proxy_cap, rng)
                Wb, J = col_id(extract(rows, cols), eps)
                blocks.append(Wb)
                Sbar[(l, tau, nu)] = cols[J]
        W_blocks[l] = blocks
    # ---- center skeleton blocks (line:extractC) ----
    B_blocks = []
    for tau in range(1 << lc):
        for nu in range(1 << (L - lc)):
            B_blocks.append(extract(Obar[(lc, tau, nu)], Sbar[(lc, tau, nu)]))
    ident_r = np.arange(m, dtype=np.int64)
    ident_c = np.arange(n, dtype=np.int64)
    return butterfly_from_blocks(L, lc, rlp, clp, ident_r, ident_c, U_blocks, R_blocks, B_blocks,
                                 W_blocks, Vt_blocks, dtype=dtype, meta=meta)


def hodbf_entry_eval(extract_user: Callable, perm: np.ndarray, leaf_ptr: np.ndarray, LH: int,
                     eps: float, proxy_cap: Optional[int] = None, seed: int = 0,
                     meta=None) -> HODBF:
    """HODBF_entry_eval: D_t = A(T_t, T_t) dense; for l = 1..LH and tau at
    level l, B_tau = A(T_tau, T_{tau^1}) by BF_entry_eval with L_B = LH - l levels
    over the sibling subtrees (L_B = 0 at l = LH)."""
    perm = np.asarray(perm, dtype=np.int64)
    lp = np.asarray(leaf_ptr, dtype=np.int64)
    n = int(lp[-1])
    D = []
    for t in range(1 << LH):
        u = perm[lp[t]:lp[t + 1]]
        D.append(extract_user(u, u))
    offdiag = []
    for l in range(1, LH + 1):
        lev = []
        w = 1 << (LH - l)
        for tau in range(1 << l):
            sib = tau ^ 1
            r0, c0 = lp[tau * w], lp[sib * w]
            rptr = lp[tau * w:(tau + 1) * w + 1] - r0
            cptr = lp[sib * w:(sib + 1) * w + 1] - c0

            def ext(I, J, r0=r0, c0=c0):
                return extract_user(perm[r0 + I], perm[c0 + J])

            lev.append(bf_entry_eval(ext, rptr, cptr, LH - l, eps, proxy_cap=proxy_cap,
                                     seed=seed + 1000 * l + tau))
        offdiag.append(lev)
    return HODBF(n, LH, lp, perm, Stage.from_blocks(D, np.complex128), offdiag, np.complex128,
                 dict(meta or {}))
