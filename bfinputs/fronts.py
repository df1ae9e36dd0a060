"""Seeded synthetic assembly trees of compressed fronts for the solve-phase sweep (SURVEY 8(f)
NEXT-4).  Input generation only: no solve arithmetic.

A complete binary assembly tree of `depth` levels (root at level 0), numbered in post-order
(children before parents, the topological order of the multifrontal sweep, Alg. 1).  Front tau
at tree level d owns the separator of a planar nx x nx grid, nx = nx_leaf + 4 (depth - d)
(the paper's fronts are planar separators), as a contiguous range of the
global unknowns.  Its update unknowns I^u_tau are a seeded subset of its parent's front
unknowns I^s_parent u I^u_parent (the extend-add containment of the multifrontal method).
  F11: the Helmholtz HOD-BF of the separator plane (10 points per wavelength, diagonal
       1 + 1j kappa h, eps 1e-4; the config-3 recipe at small size);
  F12 (s x u), F21 (u x s): random-factor butterflies with ragged ranks (L = 2, uneven leaves),
       scaled by `coupling`.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

from .configs import helmholtz_plane_hodbf
from .factors import random_ranks_butterfly


@dataclass
class Front:
    parent: int
    level: int
    s_off: int
    s_len: int
    u_idx: np.ndarray
    F11: object = None     # bfinputs.HODBF
    F12: object = None     # bfinputs.Butterfly, s x u
    F21: object = None     # bfinputs.Butterfly, u x s
    meta: dict = field(default_factory=dict)


def _split(n, parts):
    return np.array([len(a) for a in np.array_split(np.arange(n), parts)], dtype=np.int64)


def synthetic_fronts(depth: int = 2, nx_leaf: int = 8, seed: int = 0, coupling: float = 0.3,
                     u_frac: float = 0.75, dtype=np.complex128) -> (List[Front], int):
    rng = np.random.default_rng(seed)
    # post-order over a complete binary tree: node (d, i), children (d+1, 2i), (d+1, 2i+1)
    order = []

    def visit(d, i):
        if d < depth:
            visit(d + 1, 2 * i)
            visit(d + 1, 2 * i + 1)
        order.append((d, i))

    visit(0, 0)
    pos = {node: k for k, node in enumerate(order)}
    fronts: List[Front] = []
    off = 0
    for (d, i) in order:
        nx = nx_leaf + 4 * (depth - d)
        s = nx * nx
        parent = pos[(d - 1, i // 2)] if d > 0 else -1
        fronts.append(Front(parent, d, off, s, np.zeros(0, dtype=np.int64), meta={"nx": nx}))
        off += s
    N = off
    # update sets, top-down (a parent's front unknowns are known before its children's)
    for k in reversed(range(len(fronts))):
        f = fronts[k]
        if f.parent < 0:
            continue
        p = fronts[f.parent]
        pool = np.concatenate([np.arange(p.s_off, p.s_off + p.s_len), p.u_idx])
        u = min(len(pool), int(np.ceil(u_frac * f.s_len)))
        f.u_idx = np.sort(rng.choice(pool, u, replace=False)).astype(np.int64)
    for k, f in enumerate(fronts):
        H = helmholtz_plane_hodbf(f.meta["nx"], 16, 10.0, 1e-4)
        f.F11 = H if dtype == np.complex128 else H.astype(dtype)
        u = len(f.u_idx)
        if u:
            L = 2
            a = random_ranks_butterfly(L, _split(f.s_len, 1 << L), _split(u, 1 << L), seed=seed * 1000 + 2 * k,
                                       rmin=1, rmax=8)
            b = random_ranks_butterfly(L, _split(u, 1 << L), _split(f.s_len, 1 << L), seed=seed * 1000 + 2 * k + 1,
                                       rmin=1, rmax=8)
            for bf in (a, b):
                bf.U = bf.U.astype(np.complex128)
                bf.U.data *= coupling
            f.F12 = a if dtype == np.complex128 else a.astype(dtype)
            f.F21 = b if dtype == np.complex128 else b.astype(dtype)
    return fronts, N
