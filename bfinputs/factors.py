"""Packed butterfly / HOD-BF factor containers and the seeded factor generators.

This module is the *input* side shared by the CPU oracle (``oracle/``) and the CUDA
path (``paper_2007_00202_b200``).  It holds no apply arithmetic: only storage, index
bookkeeping and the random / closed-form factor recipes.

Notation follows PAPER.md Sec. 3:
  * level l in [0, L]; a block is (tau, nu) with tau a level-l node of T_O and nu a
    level-(L-l) node of T_S, both numbered left to right (children 2x, 2x+1);
  * U^L = diag(U_tau)   -- U_tau : m_tau x r^L_{tau,0}
  * R^l, l = L-1..lc -- R_{tau,nu} : (r^{l+1}_{2tau,nu>>1}+r^{l+1}_{2tau+1,nu>>1}) x r^l_{tau,nu}
  * B^{lc}   -- B_{tau,nu} : r^{lc}_{tau,nu} x c^{lc}_{tau,nu}
  * W^l, l = 1..lc -- W_{tau,nu} : c^l_{tau,nu} x (c^{l-1}_{tau>>1,2nu}+c^{l-1}_{tau>>1,2nu+1})
  * V^0 = diag(Vt_nu)   -- Vt_nu : c^0_{0,nu} x n_nu   (stored as it multiplies)
Every level's blocks are packed column-major, one after another in canonical order
``i = tau * 2^(L-l) + nu`` (tau-major, nu-minor).  That packed layout is exactly the
C-ABI layout of ``include/bfapply.h``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


# ----------------------------------------------------------------------------------
# packed stage container
# ----------------------------------------------------------------------------------
class Stage:
    """The blocks of one factor level, packed column-major in canonical order."""

    def __init__(self, rows, cols, data):
        self.rows = np.ascontiguousarray(rows, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        sizes = self.rows * self.cols
        self.offs = np.zeros(len(sizes) + 1, dtype=np.int64)
        np.cumsum(sizes, out=self.offs[1:])
        self.data = np.ascontiguousarray(data).reshape(-1)
        if self.data.size != self.offs[-1]:
            raise ValueError(f"stage data has {self.data.size} entries, expected {self.offs[-1]}")

    @property
    def nblocks(self) -> int:
        return len(self.rows)

    def block(self, i: int) -> np.ndarray:
        """Block i as an (rows x cols) view (column-major storage)."""
        r, c, o = int(self.rows[i]), int(self.cols[i]), int(self.offs[i])
        return self.data[o:o + r * c].reshape(c, r).T

    @staticmethod
    def from_blocks(blocks: List[np.ndarray], dtype) -> "Stage":
        rows = [b.shape[0] for b in blocks]
        cols = [b.shape[1] for b in blocks]
        if len(blocks) == 0:
            return Stage(rows, cols, np.zeros(0, dtype=dtype))
        data = np.concatenate([np.asarray(b, dtype=dtype).ravel(order="F") for b in blocks])
        return Stage(rows, cols, data)

    @staticmethod
    def uniform(nblocks: int, rows: int, cols: int, data: np.ndarray) -> "Stage":
        """data holds nblocks column-major (rows x cols) blocks back to back."""
        return Stage(np.full(nblocks, rows), np.full(nblocks, cols), data)

    def astype(self, dtype) -> "Stage":
        return Stage(self.rows, self.cols, self.data.astype(dtype))


@dataclass
class Butterfly:
    """Factors of Eq. (3.3) in packed canonical order.

    ``row_perm[p]`` / ``col_perm[q]`` map a tree position to the user index, so that
    K_user[row_perm[i], col_perm[j]] = K_tree[i, j].  ``R[k]`` is level l = lc + k,
    ``W[k]`` is level l = k + 1.
    """

    m: int
    n: int
    L: int
    lc: int
    row_leaf_ptr: np.ndarray
    col_leaf_ptr: np.ndarray
    row_perm: np.ndarray
    col_perm: np.ndarray
    U: Stage
    R: List[Stage]
    B: Stage
    W: List[Stage]
    Vt: Stage
    dtype: type = np.complex128
    meta: dict = field(default_factory=dict)

    # ---- canonical block index -------------------------------------------------
    def idx(self, l: int, tau: int, nu: int) -> int:
        return tau * (1 << (self.L - l)) + nu

    # ---- block accessors (views) ------------------------------------------------
    def Ub(self, tau):
        return self.U.block(tau)

    def Rb(self, l, tau, nu):
        return self.R[l - self.lc].block(self.idx(l, tau, nu))

    def Bb(self, tau, nu):
        return self.B.block(self.idx(self.lc, tau, nu))

    def Wb(self, l, tau, nu):
        return self.W[l - 1].block(self.idx(l, tau, nu))

    def Vtb(self, nu):
        return self.Vt.block(nu)

    # ---- ranks ------------------------------------------------------------------
    def rank_row(self) -> np.ndarray:
        """r^l_{tau,nu} for l = lc..L, tau-major nu-minor (C-ABI ``rank_row``)."""
        parts = [self.R[k].cols for k in range(self.L - self.lc)] + [self.U.cols]
        return np.concatenate(parts).astype(np.int32)

    def rank_col(self) -> np.ndarray:
        """c^l_{tau,nu} for l = 0..lc, tau-major nu-minor (C-ABI ``rank_col``)."""
        parts = [self.Vt.rows] + [self.W[k].rows for k in range(self.lc)]
        return np.concatenate(parts).astype(np.int32)

    def nnz(self) -> int:
        """Number of stored factor entries (U, R, B, W, Vt)."""
        tot = self.U.data.size + self.B.data.size + self.Vt.data.size
        tot += sum(s.data.size for s in self.R) + sum(s.data.size for s in self.W)
        return int(tot)

    def astype(self, dtype) -> "Butterfly":
        return Butterfly(self.m, self.n, self.L, self.lc, self.row_leaf_ptr, self.col_leaf_ptr,
                         self.row_perm, self.col_perm, self.U.astype(dtype),
                         [s.astype(dtype) for s in self.R], self.B.astype(dtype),
                         [s.astype(dtype) for s in self.W], self.Vt.astype(dtype), dtype,
                         dict(self.meta))


@dataclass
class HODBF:
    """HOD-BF matrix: dense leaf diagonals D_t plus, for every level
    l = 1..LH and node tau at level l, the butterfly of A(T_tau, T_{tau^1}).

    ``offdiag[l-1][tau]`` is that butterfly, with tree-local (identity) perms: its row
    space is T_tau's tree positions in order and its column space T_{tau^1}'s.
    ``perm[p]`` maps HOD-BF tree position p to the user index.
    """

    n: int
    LH: int
    leaf_ptr: np.ndarray
    perm: np.ndarray
    D: Stage
    offdiag: List[List[Butterfly]]
    dtype: type = np.complex128
    meta: dict = field(default_factory=dict)

    def node_range(self, l: int, tau: int):
        w = 1 << (self.LH - l)
        return int(self.leaf_ptr[tau * w]), int(self.leaf_ptr[(tau + 1) * w])

    def nnz(self) -> int:
        return int(self.D.data.size + sum(b.nnz() for lev in self.offdiag for b in lev))

    def astype(self, dtype) -> "HODBF":
        return HODBF(self.n, self.LH, self.leaf_ptr, self.perm, self.D.astype(dtype),
                     [[b.astype(dtype) for b in lev] for lev in self.offdiag], dtype,
                     dict(self.meta))


# ----------------------------------------------------------------------------------
# small helpers
# ----------------------------------------------------------------------------------
def bitrev(x, bits: int):
    """k-bit reversal of integer array x (rev_0 = 0)."""
    x = np.asarray(x, dtype=np.int64)
    r = np.zeros_like(x)
    for b in range(bits):
        r |= ((x >> b) & 1) << (bits - 1 - b)
    return r


def uniform_leaf_ptr(nleaves: int, leaf: int) -> np.ndarray:
    return np.arange(nleaves + 1, dtype=np.int64) * leaf


def _cgauss(rng, count: int, scale: float) -> np.ndarray:
    """`count` complex draws, all real parts then all imaginary parts."""
    g = rng.standard_normal(2 * count)
    return (g[:count] + 1j * g[count:]) * scale


def _cgauss_blocks(rng, nblocks: int, size: int, scale: float) -> np.ndarray:
    """nblocks blocks of `size` entries; within a block all real then all imaginary."""
    g = rng.standard_normal(nblocks * 2 * size).reshape(nblocks, 2, size)
    out = np.empty((nblocks, size), dtype=np.complex128)
    out.real = g[:, 0]
    out.imag = g[:, 1]
    out *= scale
    return out.reshape(-1)


# ----------------------------------------------------------------------------------
# generators
# ----------------------------------------------------------------------------------
def random_butterfly(L: int, leaf: int, r: int, seed: int, dtype=np.complex128,
                     lc: Optional[int] = None) -> Butterfly:
    """Config 1 / 5 recipe (BASELINE.json configs[0], configs[4]).

    n = m = leaf * 2^L, constant rank r, identity perms.  Entries i.i.d. complex
    Gaussian, real and imaginary parts N(0,1)/sqrt(2r).  Draw order: U (tau asc),
    R (l = lc..L-1, tau-major nu-minor), B, W (l = 1..lc), Vt (nu asc); within a block
    column-major, all real parts then all imaginary parts.  c64 = rounded c128 draw.
    """
    lc = L // 2 if lc is None else lc
    rng = np.random.default_rng(seed)
    nb = 1 << L
    n = leaf * nb
    s = 1.0 / np.sqrt(2.0 * r)
    U = Stage.uniform(nb, leaf, r, _cgauss_blocks(rng, nb, leaf * r, s))
    R = [Stage.uniform(nb, 2 * r, r, _cgauss_blocks(rng, nb, 2 * r * r, s)) for _ in range(lc, L)]
    B = Stage.uniform(nb, r, r, _cgauss_blocks(rng, nb, r * r, s))
    W = [Stage.uniform(nb, r, 2 * r, _cgauss_blocks(rng, nb, 2 * r * r, s)) for _ in range(1, lc + 1)]
    Vt = Stage.uniform(nb, r, leaf, _cgauss_blocks(rng, nb, r * leaf, s))
    lp = uniform_leaf_ptr(nb, leaf)
    ident = np.arange(n, dtype=np.int64)
    bf = Butterfly(n, n, L, lc, lp, lp.copy(), ident, ident.copy(), U, R, B, W, Vt,
                   np.complex128, {"kind": "random", "seed": seed, "r": r, "leaf": leaf})
    return bf if dtype == np.complex128 else bf.astype(dtype)


def random_rhs(n: int, nrhs: int, seed: int, dtype=np.complex128, rng=None) -> np.ndarray:
    """n x nrhs complex Gaussian block, std 1/sqrt(2) per part.

    Returned as an (n, nrhs) Fortran-ordered array, i.e. the column-major ABI layout
    (equivalently a C-contiguous (nrhs, n) array transposed).  Draw order: all real
    parts column-major, then all imaginary parts.
    """
    rng = np.random.default_rng(seed) if rng is None else rng
    x = _cgauss(rng, n * nrhs, 1.0 / np.sqrt(2.0)).reshape(nrhs, n)
    return np.asarray(x.T, dtype=dtype)


def random_ranks_butterfly(L: int, leaf_sizes_row, leaf_sizes_col, seed: int,
                           rmin: int = 1, rmax: int = 8, lc: Optional[int] = None,
                           dtype=np.complex128, rank_rng_seed: Optional[int] = None) -> Butterfly:
    """Random butterfly with ragged (per-block) ranks and uneven leaves.

    Used for the ragged parity cases.  Ranks r^l_{tau,nu}, c^l_{tau,nu} are drawn
    uniformly in [rmin, rmax]; block shapes then follow the rank chains of A5.
    """
    lc = L // 2 if lc is None else lc
    nb = 1 << L
    rr = np.random.default_rng(seed + 7919 if rank_rng_seed is None else rank_rng_seed)
    rng = np.random.default_rng(seed)
    row_sizes = np.asarray(leaf_sizes_row, dtype=np.int64)
    col_sizes = np.asarray(leaf_sizes_col, dtype=np.int64)
    assert len(row_sizes) == nb and len(col_sizes) == nb
    rrow = {l: rr.integers(rmin, rmax + 1, size=nb) for l in range(lc, L + 1)}
    rcol = {l: rr.integers(rmin, rmax + 1, size=nb) for l in range(0, lc + 1)}

    def idx(l, tau, nu):
        return tau * (1 << (L - l)) + nu

    def draw(shape):
        return _cgauss(rng, shape[0] * shape[1], 1.0).reshape(shape[1], shape[0]).T / np.sqrt(max(shape[1], 1))

    U = [draw((int(row_sizes[t]), int(rrow[L][t]))) for t in range(nb)]
    R = []
    for l in range(lc, L):
        blocks = []
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                ra = rrow[l + 1][idx(l + 1, 2 * tau, nu >> 1)]
                rb = rrow[l + 1][idx(l + 1, 2 * tau + 1, nu >> 1)]
                blocks.append(draw((int(ra + rb), int(rrow[l][idx(l, tau, nu)]))))
        R.append(Stage.from_blocks(blocks, np.complex128))
    B = [draw((int(rrow[lc][i]), int(rcol[lc][i]))) for i in range(nb)]
    W = []
    for l in range(1, lc + 1):
        blocks = []
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                ca = rcol[l - 1][idx(l - 1, tau >> 1, 2 * nu)]
                cb = rcol[l - 1][idx(l - 1, tau >> 1, 2 * nu + 1)]
                blocks.append(draw((int(rcol[l][idx(l, tau, nu)]), int(ca + cb))))
        W.append(Stage.from_blocks(blocks, np.complex128))
    Vt = [draw((int(rcol[0][nu]), int(col_sizes[nu]))) for nu in range(nb)]
    rlp = np.concatenate([[0], np.cumsum(row_sizes)]).astype(np.int64)
    clp = np.concatenate([[0], np.cumsum(col_sizes)]).astype(np.int64)
    m, n = int(rlp[-1]), int(clp[-1])
    prow = np.random.default_rng(seed + 1).permutation(m).astype(np.int64)
    pcol = np.random.default_rng(seed + 2).permutation(n).astype(np.int64)
    bf = Butterfly(m, n, L, lc, rlp, clp, prow, pcol,
                   Stage.from_blocks(U, np.complex128), R, Stage.from_blocks(B, np.complex128), W,
                   Stage.from_blocks(Vt, np.complex128), np.complex128,
                   {"kind": "ragged", "seed": seed})
    return bf if dtype == np.complex128 else bf.astype(dtype)


def identity_butterfly(L: int, m0: int, dtype=np.complex128) -> Butterfly:
    """Closed-form identity butterfly (pin P1).

    n = m0 * 2^L, rank m0; T_S leaf q covers user columns [rev_L(q) m0, +m0) and the
    row tree is in natural order.  U = Vt = B = I, R_{tau,nu} = [I;0] (nu even) or
    [0;I] (nu odd), W_{tau,nu} = [I,0] (tau even) or [0,I] (tau odd).  Then K = I.
    """
    lc = L // 2
    nb = 1 << L
    n = m0 * nb
    I = np.eye(m0)
    Z = np.zeros((m0, m0))
    U = Stage.from_blocks([I] * nb, np.complex128)
    Vt = Stage.from_blocks([I] * nb, np.complex128)
    B = Stage.from_blocks([I] * nb, np.complex128)
    R = []
    for l in range(lc, L):
        blocks = []
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                blocks.append(np.vstack([I, Z]) if nu % 2 == 0 else np.vstack([Z, I]))
        R.append(Stage.from_blocks(blocks, np.complex128))
    W = []
    for l in range(1, lc + 1):
        blocks = []
        for tau in range(1 << l):
            for nu in range(1 << (L - l)):
                blocks.append(np.hstack([I, Z]) if tau % 2 == 0 else np.hstack([Z, I]))
        W.append(Stage.from_blocks(blocks, np.complex128))
    lp = uniform_leaf_ptr(nb, m0)
    q = np.arange(n) // m0
    col_perm = (bitrev(q, L) * m0 + np.arange(n) % m0).astype(np.int64)
    bf = Butterfly(n, n, L, lc, lp, lp.copy(), np.arange(n, dtype=np.int64), col_perm,
                   U, R, B, W, Vt, np.complex128, {"kind": "identity", "m0": m0})
    return bf if dtype == np.complex128 else bf.astype(dtype)


def dft_butterfly(L: int, dtype=np.complex128) -> Butterfly:
    """Closed-form DFT butterfly, leaf 1, rank 1 (pin P3).

    n = 2^L, omega = exp(-2 pi i / n), row_perm[p] = rev_L(p), col_perm[q] = rev_L(q):
      B_{tau,nu}  = omega^(-rev_lc(tau) rev_{L-lc}(nu))
      R_{tau,nu}  = [omega^(rev_{l+1}(2tau) d); omega^(rev_{l+1}(2tau+1) d)],
                    d = rev_{L-l}(nu) - rev_{L-l-1}(nu>>1)          (l = lc..L-1)
      W_{tau,nu}  = [omega^(e rev_{L-l+1}(2nu)), omega^(e rev_{L-l+1}(2nu+1))],
                    e = rev_l(tau) - rev_{l-1}(tau>>1)               (l = 1..lc)
    Then K_user = F with F_jk = omega^(jk).  Exponents are reduced mod n in integers
    before exp() so the twiddles stay accurate at n = 2^20.
    """
    lc = L // 2
    n = 1 << L
    nb = n

    def tw(e):
        e = np.mod(np.asarray(e, dtype=np.int64), n)
        return np.exp(-2j * np.pi * e.astype(np.float64) / n)

    one = np.ones(nb, dtype=np.complex128)
    U = Stage.uniform(nb, 1, 1, one)
    Vt = Stage.uniform(nb, 1, 1, one.copy())
    i = np.arange(nb, dtype=np.int64)
    tau_c, nu_c = i >> (L - lc), i & ((1 << (L - lc)) - 1)
    B = Stage.uniform(nb, 1, 1, tw(-bitrev(tau_c, lc) * bitrev(nu_c, L - lc)))
    R = []
    for l in range(lc, L):
        tau, nu = i >> (L - l), i & ((1 << (L - l)) - 1)
        d = bitrev(nu, L - l) - bitrev(nu >> 1, L - l - 1)
        top = tw(bitrev(2 * tau, l + 1) * d)
        bot = tw(bitrev(2 * tau + 1, l + 1) * d)
        R.append(Stage.uniform(nb, 2, 1, np.stack([top, bot], axis=1).reshape(-1)))
    W = []
    for l in range(1, lc + 1):
        tau, nu = i >> (L - l), i & ((1 << (L - l)) - 1)
        e = bitrev(tau, l) - bitrev(tau >> 1, l - 1)
        left = tw(e * bitrev(2 * nu, L - l + 1))
        right = tw(e * bitrev(2 * nu + 1, L - l + 1))
        # (1 x 2) block, column-major: [left, right]
        W.append(Stage.uniform(nb, 1, 2, np.stack([left, right], axis=1).reshape(-1)))
    lp = uniform_leaf_ptr(nb, 1)
    perm = bitrev(np.arange(n), L)
    bf = Butterfly(n, n, L, lc, lp, lp.copy(), perm, perm.copy(), U, R, B, W, Vt,
                   np.complex128, {"kind": "dft"})
    return bf if dtype == np.complex128 else bf.astype(dtype)


def butterfly_from_blocks(L, lc, row_leaf_ptr, col_leaf_ptr, row_perm, col_perm,
                          U, R, B, W, Vt, dtype=np.complex128, meta=None) -> Butterfly:
    """Pack per-block lists (U[tau], R[l][idx], B[idx], W[l][idx], Vt[nu]) into a Butterfly.

    R is a dict/list indexed by level l (lc..L-1), W by level l (1..lc); each holds the
    level's blocks in canonical order.
    """
    rlp = np.asarray(row_leaf_ptr, dtype=np.int64)
    clp = np.asarray(col_leaf_ptr, dtype=np.int64)
    return Butterfly(int(rlp[-1]), int(clp[-1]), L, lc, rlp, clp,
                     np.asarray(row_perm, dtype=np.int64), np.asarray(col_perm, dtype=np.int64),
                     Stage.from_blocks(U, dtype), [Stage.from_blocks(R[l], dtype) for l in range(lc, L)],
                     Stage.from_blocks(B, dtype), [Stage.from_blocks(W[l], dtype) for l in range(1, lc + 1)],
                     Stage.from_blocks(Vt, dtype), dtype, dict(meta or {}))


# ----------------------------------------------------------------------------------
# non-canonical block orderings (C-ABI bf_desc.level_maps; layout only, no arithmetic)
# ----------------------------------------------------------------------------------
def random_level_maps(L: int, seed: int, levels=None) -> list:
    """L + 1 entries: a seeded random bijection of [0, 2^L) for every level in ``levels``
    (default: all), None (canonical) for the others."""
    rng = np.random.default_rng(seed)
    nb = 1 << L
    levels = range(L + 1) if levels is None else levels
    return [rng.permutation(nb).astype(np.int32) if l in levels else None for l in range(L + 1)]


def slot_ordered(bf: Butterfly, maps) -> Butterfly:
    """The same butterfly with the blocks (and hence the ranks) of every mapped level packed in
    storage-slot order: slot s of level l holds canonical block maps[l][s]."""
    def perm(stage: Stage, mp) -> Stage:
        if mp is None:
            return stage
        return Stage.from_blocks([stage.block(int(i)) for i in mp], bf.dtype)

    L, lc = bf.L, bf.lc
    return Butterfly(bf.m, bf.n, L, lc, bf.row_leaf_ptr, bf.col_leaf_ptr, bf.row_perm, bf.col_perm,
                     perm(bf.U, maps[L]), [perm(s, maps[lc + k]) for k, s in enumerate(bf.R)],
                     perm(bf.B, maps[lc]), [perm(s, maps[k + 1]) for k, s in enumerate(bf.W)],
                     perm(bf.Vt, maps[0]), bf.dtype, dict(bf.meta))
