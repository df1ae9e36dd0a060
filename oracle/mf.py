"""CPU oracle of the multifrontal solve-phase sweep -- TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's cpu legs.  Follows P:697
(Alg. 1 line precGMRES) in the paper's order, with every front densified by oracle.dense:
  forward, leaves to root:   z_s = F11^{-1} y_s  (a dense solve);  y_u -= F21 z_s
  backward, root to leaves:  x_s = z_s - F11^{-1} (F12 x_u)
Pinned in tests/test_oracle_mf.py: with F12 = F21 = 0 the sweep is the block-diagonal solve; on
a two-front tree it equals the dense solve of the assembled block-LU matrix.
"""
from __future__ import annotations

import numpy as np

from .dense import bf_dense, hodbf_dense


def mf_solve(fronts, N, B):
    B = np.asarray(B, dtype=np.complex128)
    y = B.copy()
    x = np.zeros_like(B)
    F11 = [hodbf_dense(f.F11) for f in fronts]
    for k, f in enumerate(fronts):                       # post-order: children first
        s = slice(f.s_off, f.s_off + f.s_len)
        x[s] = np.linalg.solve(F11[k], y[s])
        if len(f.u_idx):
            y[f.u_idx] -= bf_dense(f.F21) @ x[s]
    for k in reversed(range(len(fronts))):               # root first
        f = fronts[k]
        if not len(f.u_idx):
            continue
        s = slice(f.s_off, f.s_off + f.s_len)
        x[s] -= np.linalg.solve(F11[k], bf_dense(f.F12) @ x[f.u_idx])
    return x


def mf_matrix(fronts, N):
    """M with M^{-1} = the sweep: M = L U, L = I + sum_tau (blocks F11 - I on (s, s) and F21 on (u, s)),
    U = I + sum_tau F11^{-1} F12 on (s, u) -- the block LU of the fronts, assembled densely (for pins)."""
    L = np.eye(N, dtype=np.complex128)
    U = np.eye(N, dtype=np.complex128)
    for f in fronts:
        s = np.arange(f.s_off, f.s_off + f.s_len)
        A11 = hodbf_dense(f.F11)
        L[np.ix_(s, s)] = A11
        if len(f.u_idx):
            L[np.ix_(f.u_idx, s)] = bf_dense(f.F21)
            U[np.ix_(s, f.u_idx)] = np.linalg.solve(A11, bf_dense(f.F12))
    return L @ U
