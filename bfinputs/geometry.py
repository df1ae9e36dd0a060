"""Synthetic separator-front geometry and kernels for BASELINE.json configs 2-4.

Readings (DESIGN.md / SURVEY C4):
  A12  h = 1; grid point (i, j) sits at (i h, j h, z); user index i + nx j.  Config 2's
       second plane is at z = 8h, aligned.  kappa = 2 pi / (ppw h).  Trees: recursive
       bisection of the index box, splitting the longer axis (x on ties), lower half
       first, to a uniform depth.  Config 4's unknowns are point-major, component-minor
       (x then y), so both components of a point share a leaf.
  A11  self term of the scalar kernel: A_ii = 1 + 1j kappa h; config 4 applies it to the
       2x2 self block as (1 + 1j kappa h) I_2.
  A13  dyadic kernel (I + grad grad / kappa^2) g, g = e^{i kappa r} / (4 pi r); the
       in-plane 2x2 block.
These are input recipes only (no apply arithmetic).
"""
from __future__ import annotations

import numpy as np


def grid_points(nx: int, ny: int, z: float = 0.0, h: float = 1.0) -> np.ndarray:
    """(nx*ny, 3) coordinates, user index i + nx*j."""
    j, i = np.divmod(np.arange(nx * ny), nx)
    return np.stack([i * h, j * h, np.full(nx * ny, z)], axis=1).astype(np.float64)


def bisection_tree(nx: int, ny: int, depth: int):
    """Recursive bisection of the (nx x ny) index box to `depth` levels.

    Returns (perm, leaf_ptr): perm[p] = user point index (i + nx j) at tree position p;
    leaf_ptr has 2^depth + 1 offsets.  Split the longer axis (x on ties), lower half
    first; points inside a leaf box are ordered by user index.
    """
    boxes = [(0, nx, 0, ny)]
    for _ in range(depth):
        nxt = []
        for (x0, x1, y0, y1) in boxes:
            if (x1 - x0) >= (y1 - y0):
                xm = x0 + (x1 - x0) // 2
                nxt += [(x0, xm, y0, y1), (xm, x1, y0, y1)]
            else:
                ym = y0 + (y1 - y0) // 2
                nxt += [(x0, x1, y0, ym), (x0, x1, ym, y1)]
        boxes = nxt
    perm, ptr = [], [0]
    for (x0, x1, y0, y1) in boxes:
        jj, ii = np.meshgrid(np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
        idx = (ii + nx * jj).reshape(-1)
        perm.append(np.sort(idx))
        ptr.append(ptr[-1] + idx.size)
    return np.concatenate(perm).astype(np.int64), np.asarray(ptr, dtype=np.int64)


def tree_depth_for_leaf(npts: int, leaf: int) -> int:
    d = 0
    while (npts >> d) > leaf:
        d += 1
    return d


def expand_components(perm_pts: np.ndarray, ptr_pts: np.ndarray, ncomp: int):
    """Point tree -> unknown tree for point-major, component-minor unknowns."""
    perm = (perm_pts[:, None] * ncomp + np.arange(ncomp)[None, :]).reshape(-1)
    return perm.astype(np.int64), (ptr_pts * ncomp).astype(np.int64)


def helmholtz(P: np.ndarray, Q: np.ndarray, kappa: float, self_value=None) -> np.ndarray:
    """G(p, q) = exp(i kappa |p-q|) / (4 pi |p-q|); entries with p == q get self_value."""
    d = P[:, None, :] - Q[None, :, :]
    r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
    zero = r == 0.0
    rs = np.where(zero, 1.0, r)
    G = np.exp(1j * kappa * rs) / (4.0 * np.pi * rs)
    if zero.any():
        if self_value is None:
            raise ValueError("coincident points but no self_value")
        G[zero] = self_value
    return G


def dyadic(P: np.ndarray, Q: np.ndarray, kappa: float, self_value=None) -> np.ndarray:
    """In-plane (x, y) 2x2 blocks of the dyadic Green's function.

    Gbar = g(r) [(1 + i/(kr) - 1/(kr)^2) I + (3/(kr)^2 - 3i/(kr) - 1) rhat rhat^T].
    Returns a (2|P| x 2|Q|) matrix, point-major component-minor.  Coincident points
    get self_value * I_2.
    """
    d = P[:, None, :] - Q[None, :, :]
    r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
    zero = r == 0.0
    rs = np.where(zero, 1.0, r)
    kr = kappa * rs
    g = np.exp(1j * kr) / (4.0 * np.pi * rs)
    a = g * (1.0 + 1j / kr - 1.0 / kr ** 2)
    b = g * (3.0 / kr ** 2 - 3j / kr - 1.0)
    rh = d / rs[:, :, None]
    out = np.empty((P.shape[0], 2, Q.shape[0], 2), dtype=np.complex128)
    for s in range(2):
        for t in range(2):
            out[:, s, :, t] = b * rh[:, :, s] * rh[:, :, t] + (a if s == t else 0.0)
    if zero.any():
        if self_value is None:
            raise ValueError("coincident points but no self_value")
        for s in range(2):
            for t in range(2):
                out[:, s, :, t][zero] = self_value if s == t else 0.0
    return out.reshape(2 * P.shape[0], 2 * Q.shape[0])


class KernelMatrix:
    """Entry oracle A(i, j) over user indices for a point-kernel pair (extract())."""

    def __init__(self, P_rows, P_cols, kappa, kind="helmholtz", self_value=None):
        self.P_rows, self.P_cols, self.kappa = P_rows, P_cols, kappa
        self.kind, self.self_value = kind, self_value
        self.ncomp = 2 if kind == "dyadic" else 1
        self.shape = (P_rows.shape[0] * self.ncomp, P_cols.shape[0] * self.ncomp)

    def __call__(self, I, J) -> np.ndarray:
        I = np.asarray(I, dtype=np.int64)
        J = np.asarray(J, dtype=np.int64)
        if self.kind == "helmholtz":
            return helmholtz(self.P_rows[I], self.P_cols[J], self.kappa, self.self_value)
        # dyadic: evaluate per unique point then select components
        pi, ci = np.divmod(I, 2)
        pj, cj = np.divmod(J, 2)
        upi, inv_i = np.unique(pi, return_inverse=True)
        upj, inv_j = np.unique(pj, return_inverse=True)
        G = dyadic(self.P_rows[upi], self.P_cols[upj], self.kappa, self.self_value)
        return G[(2 * inv_i + ci)[:, None], (2 * inv_j + cj)[None, :]]
