"""Binding of the randomized matrix-free construction (bf_random_matvec, include/bfapply.h;
PAPER.md Sec. 3.3) and of composite operators (bf_operator_apply).

Argument marshalling only: the sketches, the batched interpolative decompositions and the centre
solves run in libbfapply's kernels; the operator is applied by the library (bf_operator_apply)
or by a Python callable that itself calls library applies.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from .bfapply import (BF_C128, BF_C64, OPS, BFHandle, HODBFHandle, _check, _i64p, _np_dtype_code, _ptr,
                      _torch_dtype, lib)

(BF_FACTOR_BF, BF_FACTOR_HODBF, BF_FACTOR_IDENTITY, BF_FACTOR_BF_PLUS_I, BF_FACTOR_SELECT, BF_FACTOR_HODBF_INV,
 BF_FACTOR_HODBF_INV_NODE) = range(7)

MATVEC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                        C.c_void_p)


class bf_rmv_desc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("L", C.c_int32), ("lc", C.c_int32), ("rank_max", C.c_int32),
                ("m", C.c_int64), ("n", C.c_int64),
                ("row_leaf_ptr", _i64p), ("col_leaf_ptr", _i64p), ("row_perm", _i64p), ("col_perm", _i64p),
                ("eps", C.c_double), ("oversample", C.c_int32), ("reserved", C.c_int32),
                ("seed", C.c_uint64), ("chunk_bytes", C.c_size_t)]


class bf_rmv_stats(C.Structure):
    _fields_ = [("matvec_cols_n", C.c_int64), ("matvec_cols_c", C.c_int64), ("max_rank", C.c_int32),
                ("saturated", C.c_int32), ("t_matvec_ms", C.c_double), ("t_total_ms", C.c_double)]


class bf_factor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("op", C.c_int32), ("handle", C.c_void_p), ("rows", C.c_int64),
                ("cols", C.c_int64), ("aux0", C.c_int64), ("aux1", C.c_int64)]


class bf_inv_opts(C.Structure):
    _fields_ = [("eps", C.c_double), ("rank_max", C.c_int32), ("oversample", C.c_int32), ("seed", C.c_uint64),
                ("dense_max", C.c_int64)]


class bf_product(C.Structure):
    _fields_ = [("alpha_re", C.c_double), ("alpha_im", C.c_double), ("nfac", C.c_int32), ("reserved", C.c_int32),
                ("fac", C.POINTER(bf_factor)), ("row_off", C.c_int64), ("col_off", C.c_int64)]


class bf_operator(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("nprod", C.c_int32), ("m", C.c_int64), ("n", C.c_int64),
                ("prod", C.POINTER(bf_product))]


_registered = False


def _lib():
    global _registered
    L = lib()
    if not _registered:
        L.bf_random_matvec.restype = C.c_int
        L.bf_random_matvec.argtypes = [C.POINTER(bf_rmv_desc), C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                       C.POINTER(C.c_void_p), C.POINTER(bf_rmv_stats)]
        L.bf_operator_apply.restype = C.c_int
        L.bf_operator_apply.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_int64, C.c_void_p]
        L.bf_batched_id.restype = C.c_int
        L.bf_batched_id.argtypes = [C.c_int, C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.c_void_p, C.c_double,
                                    C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.hodbf_invert.restype = C.c_int
        L.hodbf_invert.argtypes = [C.c_void_p, C.POINTER(bf_inv_opts), C.c_int, C.c_void_p, C.POINTER(C.c_void_p),
                                   C.POINTER(bf_rmv_stats)]
        L.hodbf_inv_destroy.restype = C.c_int
        L.hodbf_inv_destroy.argtypes = [C.c_void_p]
        L.hodbf_inv_apply.restype = C.c_int
        L.hodbf_inv_apply.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_size_t, C.c_void_p]
        L.hodbf_inv_workspace_size.restype = C.c_int
        L.hodbf_inv_workspace_size.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_size_t)]
        L.hodbf_inv_info.restype = C.c_int
        L.hodbf_inv_info.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.bf_export.restype = C.c_int
        L.bf_export.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _registered = True
    return L


Factor = Union[Tuple[object, str], Tuple[str, int]]


class Operator:
    """A = sum_s alpha_s P_s with P_s = f_{q-1} ... f_0 (f_0 applied first), each placed at
    (row_off, col_off) inside the m x n operator.  A factor is (handle, "N" | "C") for a
    BFHandle / HODBFHandle / HODBFInverse, ("I", size) or ("I+", K) for I + K.  Applied by the
    library (bf_operator_apply)."""

    def __init__(self, m: int, n: int, dtype, products: Sequence[Tuple[complex, Sequence[Factor], int, int]]):
        self.m, self.n = m, n
        self.code = _np_dtype_code(dtype)
        self._keep = []
        prods = (bf_product * len(products))()
        for s, (alpha, facs, ro, co) in enumerate(products):
            arr = (bf_factor * len(facs))()
            for q, f in enumerate(facs):
                a = arr[q]
                if f[0] == "I":
                    a.kind, a.op, a.handle, a.rows, a.cols = BF_FACTOR_IDENTITY, OPS["N"], None, f[1], f[1]
                    continue
                if f[0] == "I+":  # ("I+", K): I + K for a square butterfly handle
                    a.kind, a.op, a.handle, a.rows, a.cols = BF_FACTOR_BF_PLUS_I, OPS["N"], f[1].h, f[1].m, f[1].m
                    self._keep.append(f[1])
                    continue
                h, op = f
                self._keep.append(h)
                if isinstance(h, HODBFHandle):
                    a.kind, rows, cols = BF_FACTOR_HODBF, h.n, h.n
                elif isinstance(h, HODBFInverse):
                    a.kind, rows, cols = BF_FACTOR_HODBF_INV, h.n, h.n
                else:
                    a.kind, rows, cols = BF_FACTOR_BF, h.m, h.n
                a.op, a.handle = OPS[op], h.h
                a.rows, a.cols = (rows, cols) if op == "N" else (cols, rows)
            self._keep.append(arr)
            p = prods[s]
            p.alpha_re, p.alpha_im = complex(alpha).real, complex(alpha).imag
            p.nfac, p.fac, p.row_off, p.col_off = len(facs), arr, ro, co
        self._keep.append(prods)
        self.desc = bf_operator(self.code, len(products), m, n, prods)

    @property
    def ctx(self):
        return C.cast(C.pointer(self.desc), C.c_void_p)

    @property
    def fn(self):
        return C.cast(_lib().bf_operator_apply, C.c_void_p)

    def apply(self, X: torch.Tensor, op: str = "N") -> torch.Tensor:
        """Y = A X (op N) or A^H X (op C); X (nrhs, rows) on the device."""
        rin, rout = (self.n, self.m) if op == "N" else (self.m, self.n)
        assert X.is_cuda and X.dim() == 2 and X.shape[1] == rin and X.is_contiguous()
        Y = torch.empty((X.shape[0], rout), dtype=X.dtype, device=X.device)
        st = torch.cuda.current_stream()
        _check("bf_operator_apply", _lib().bf_operator_apply(self.ctx, OPS[op], X.shape[0], C.c_void_p(X.data_ptr()),
                                                              max(rin, 1), C.c_void_p(Y.data_ptr()), max(rout, 1),
                                                              C.c_void_p(st.cuda_stream)))
        return Y


class _CudaBlock:
    """A raw device block exposed to torch through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr, rows, ld, nrhs, dtype):
        self.__cuda_array_interface__ = {"shape": (nrhs, rows), "typestr": np.dtype(dtype).str,
                                         "data": (ptr, False), "version": 3,
                                         "strides": (ld * np.dtype(dtype).itemsize, np.dtype(dtype).itemsize)}


def callback(fn: Callable[[str, torch.Tensor, torch.Tensor], None], dtype):
    """Wrap fn(op, X, Y) -- X, Y torch views (nrhs, rows) of the library's device blocks; fn must
    write Y = A X (op "N") or A^H X (op "C") with library applies -- as a bf_matvec_fn."""
    npdt = np.complex128 if _np_dtype_code(dtype) == BF_C128 else np.complex64
    inv = {v: k for k, v in OPS.items()}

    def _cb(ctx, op, nrhs, X, ldx, Y, ldy, stream):
        try:
            Xt = torch.as_tensor(_CudaBlock(X, ldx, ldx, nrhs, npdt), device="cuda")
            Yt = torch.as_tensor(_CudaBlock(Y, ldy, ldy, nrhs, npdt), device="cuda")
            fn(inv[op], Xt, Yt)
            return 0
        except Exception as e:  # no exception may cross the C boundary
            print(f"bf_random_matvec callback: {e!r}")
            return -1

    return MATVEC_FN(_cb)


class RandomMatvecResult:
    def __init__(self, handle: BFHandle, stats: bf_rmv_stats, trees):
        self.handle = handle
        self.stats = {f: getattr(stats, f) for f, _ in bf_rmv_stats._fields_}
        self.trees = trees


def random_matvec(op: Union[Operator, Callable], m: int, n: int, L: int, row_leaf_ptr, col_leaf_ptr,
                  row_perm=None, col_perm=None, lc: Optional[int] = None, eps: float = 1e-10, rank_max: int = 32,
                  oversample: int = 10, seed: int = 1, dtype=np.complex128, device: int = 0,
                  chunk_bytes: int = 0) -> RandomMatvecResult:
    """BF_random_matvec(A): a butterfly with the given trees approximating the operator
    A (m x n), from products with Gaussian sketches.  `op` is an Operator (applied by the library)
    or a callable fn(op, X, Y) (see `callback`)."""
    keep = []

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a

    d = bf_rmv_desc()
    d.dtype = _np_dtype_code(dtype)
    d.L, d.lc = L, -1 if lc is None else lc
    d.rank_max, d.m, d.n = rank_max, m, n
    rlp, clp = arr(row_leaf_ptr, np.int64), arr(col_leaf_ptr, np.int64)
    d.row_leaf_ptr, d.col_leaf_ptr = _ptr(rlp, C.c_int64), _ptr(clp, C.c_int64)
    rp = None if row_perm is None else arr(row_perm, np.int64)
    cp = None if col_perm is None else arr(col_perm, np.int64)
    d.row_perm = _ptr(rp, C.c_int64) if rp is not None else None
    d.col_perm = _ptr(cp, C.c_int64) if cp is not None else None
    d.eps, d.oversample, d.seed, d.chunk_bytes = eps, oversample, seed, chunk_bytes
    if isinstance(op, Operator):
        fn, ctx = op.fn, op.ctx
    else:
        cb = callback(op, dtype)
        keep.append(cb)
        fn, ctx = C.cast(cb, C.c_void_p), None
    h = C.c_void_p()
    stats = bf_rmv_stats()
    st = torch.cuda.current_stream(device)
    _check("bf_random_matvec", _lib().bf_random_matvec(C.byref(d), fn, ctx, device, C.c_void_p(st.cuda_stream),
                                                         C.byref(h), C.byref(stats)))
    lc_v = L // 2 if lc is None else lc
    trees = {"L": L, "lc": lc_v, "m": m, "n": n, "row_leaf_ptr": rlp, "col_leaf_ptr": clp,
             "row_perm": np.arange(m) if rp is None else rp, "col_perm": np.arange(n) if cp is None else cp,
             "dtype": dtype}
    return RandomMatvecResult(BFHandle.from_raw(h, device, d.dtype, m, n), stats, trees)


def export(handle: BFHandle, trees) -> "object":
    """The handle's factors as a bfinputs.Butterfly on the host (bf_export), for host tooling and
    the CPU oracle.  `trees`: the dict RandomMatvecResult.trees (leaf offsets, perms, L, lc)."""
    from bfinputs.factors import Butterfly, Stage
    L, lc, m, n = trees["L"], trees["lc"], trees["m"], trees["n"]
    nb = 1 << L
    lens = (C.c_int64 * 5)()
    rr = np.zeros((L - lc + 1) * nb, dtype=np.int32)
    rcn = np.zeros((lc + 1) * nb, dtype=np.int32)
    L_ = _lib()
    _check("bf_export", L_.bf_export(handle.h, lens, rr.ctypes.data_as(C.POINTER(C.c_int32)),
                                     rcn.ctypes.data_as(C.POINTER(C.c_int32)), None, None, None, None, None))
    cdt = np.complex128 if handle.code == BF_C128 else np.complex64
    bufs = [np.zeros(lens[q], dtype=cdt) for q in range(5)]
    _check("bf_export", L_.bf_export(handle.h, lens, None, None, *[_ptr(b) for b in bufs]))
    U, Rall, Bd, Wall, Vtd = bufs
    r = rr.reshape(L - lc + 1, nb)
    c = rcn.reshape(lc + 1, nb)
    rlp, clp = trees["row_leaf_ptr"], trees["col_leaf_ptr"]
    idx = lambda l, t, v: (t << (L - l)) | v  # noqa: E731
    Ust = Stage(np.diff(rlp), r[L - lc], U)
    Rs, o = [], 0
    for l in range(lc, L):
        rows = np.array([r[l + 1 - lc][idx(l + 1, 2 * (i >> (L - l)), (i & ((1 << (L - l)) - 1)) >> 1)] +
                         r[l + 1 - lc][idx(l + 1, 2 * (i >> (L - l)) + 1, (i & ((1 << (L - l)) - 1)) >> 1)]
                         for i in range(nb)], dtype=np.int64)
        cols = r[l - lc].astype(np.int64)
        sz = int((rows * cols).sum())
        Rs.append(Stage(rows, cols, Rall[o:o + sz]))
        o += sz
    Bst = Stage(r[0], c[lc], Bd)
    Ws, o = [], 0
    for l in range(1, lc + 1):
        rows = c[l].astype(np.int64)
        cols = np.array([c[l - 1][idx(l - 1, (i >> (L - l)) >> 1, 2 * (i & ((1 << (L - l)) - 1)))] +
                         c[l - 1][idx(l - 1, (i >> (L - l)) >> 1, 2 * (i & ((1 << (L - l)) - 1)) + 1)]
                         for i in range(nb)], dtype=np.int64)
        sz = int((rows * cols).sum())
        Ws.append(Stage(rows, cols, Wall[o:o + sz]))
        o += sz
    Vst = Stage(c[0], np.diff(clp), Vtd)
    return Butterfly(m, n, L, lc, np.asarray(rlp, np.int64), np.asarray(clp, np.int64),
                     np.asarray(trees["row_perm"], np.int64), np.asarray(trees["col_perm"], np.int64),
                     Ust, Rs, Bst, Ws, Vst, cdt, {"kind": "random_matvec"})


def batched_id(mats: Sequence[torch.Tensor], eps: float, rmax: int):
    """bf_batched_id on a list of (k x p_i) complex device matrices (given as torch tensors of
    shape (p_i, k), i.e. column-major k x p_i).  Returns [(rank, perm, T)] with T = R11^{-1} R12
    (rank x (p_i - rank))."""
    k = mats[0].shape[1]
    assert all(m.shape[1] == k for m in mats), "one sketch width k per call"
    dt = mats[0].dtype
    flat = torch.cat([m.reshape(-1) for m in mats]).contiguous()
    pc = np.array([m.shape[0] for m in mats], dtype=np.int64)
    rank = torch.zeros(len(mats), dtype=torch.int32, device=flat.device)
    perm = torch.zeros(max(int(pc.sum()), 1), dtype=torch.int32, device=flat.device)
    code = BF_C128 if dt == torch.complex128 else BF_C64
    st = torch.cuda.current_stream()
    _check("bf_batched_id", _lib().bf_batched_id(code, len(mats), k, pc.ctypes.data_as(C.POINTER(C.c_int64)),
                                                 C.c_void_p(flat.data_ptr()), eps, rmax,
                                                 C.c_void_p(rank.data_ptr()), C.c_void_p(perm.data_ptr()),
                                                 C.c_void_p(st.cuda_stream)))
    out, o, po = [], 0, 0
    rk, pm, F = rank.cpu().numpy(), perm.cpu().numpy(), flat.cpu().numpy()
    for i, p in enumerate(pc):
        A = F[o:o + p * k].reshape(p, k).T  # k x p
        r = int(rk[i])
        out.append((r, pm[po:po + p].copy(), A[:r, r:].copy()))
        o += p * k
        po += p
    return out


class HODBFInverse:
    """A^{-1} of an HOD-BF matrix built by hodbf_invert (Alg. 4 HODBF_invert with BF_SMW,
    P:569-615): dense leaf inverses and one butterfly per internal node, applied as their
    product (include/bfapply.h)."""

    def __init__(self, H, eps: float = 1e-10, rank_max: int = 64, oversample: int = 10, seed: int = 1,
                 dense_max: int = 0, device: int = 0):
        from .bfapply import _Keep, make_hodbf_desc
        keep = _Keep()
        d = make_hodbf_desc(H, keep)
        code = d.dtype
        o = bf_inv_opts(eps, rank_max, oversample, seed, dense_max)
        h = C.c_void_p()
        st = bf_rmv_stats()
        cs = torch.cuda.current_stream(device)
        _check("hodbf_invert", _lib().hodbf_invert(C.byref(d), C.byref(o), device, C.c_void_p(cs.cuda_stream),
                                                     C.byref(h), C.byref(st)))
        self.h, self.n, self.code, self.device = h, H.n, code, device
        self.stats = {f: getattr(st, f) for f, _ in bf_rmv_stats._fields_}
        fe, nb = C.c_int64(), C.c_int32()
        _check("hodbf_inv_info", _lib().hodbf_inv_info(h, C.byref(fe), C.byref(nb)))
        self.factor_entries, self.nbutterflies = fe.value, nb.value

    def close(self):
        if getattr(self, "h", None):
            _lib().hodbf_inv_destroy(self.h)
            self.h = None

    __del__ = close

    def apply(self, X: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Y = A^{-1} X (op N) or A^{-H} X (op C); X (nrhs, n) on the device."""
        assert X.is_cuda and X.dim() == 2 and X.shape[1] == self.n and X.stride(1) == 1
        if out is None:
            out = torch.empty((X.shape[0], self.n), dtype=X.dtype, device=X.device)
        st = torch.cuda.current_stream()
        ws = C.c_size_t()
        _check("hodbf_inv_workspace_size", _lib().hodbf_inv_workspace_size(self.h, X.shape[0], C.byref(ws)))
        work = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=X.device)
        _check("hodbf_inv_apply", _lib().hodbf_inv_apply(self.h, OPS[op], X.shape[0], C.c_void_p(X.data_ptr()),
                                                          max(X.stride(0), self.n, 1), C.c_void_p(out.data_ptr()),
                                                          max(out.stride(0), self.n, 1), C.c_void_p(work.data_ptr()),
                                                          work.numel(), C.c_void_p(st.cuda_stream)))
        return out


class bf_front(C.Structure):
    _fields_ = [("parent", C.c_int32), ("reserved", C.c_int32), ("s_off", C.c_int64), ("s_len", C.c_int64),
                ("u_len", C.c_int64), ("u_idx", C.POINTER(C.c_int64)), ("F11inv", C.c_void_p), ("F12", C.c_void_p),
                ("F21", C.c_void_p)]


class MFSolver:
    """The multifrontal solve-phase sweep (bf_mf_solve) over an assembly tree of fronts
    (bfinputs.fronts.Front: F11 HOD-BF, F12 / F21 butterflies, separator range, update indices).
    Builds every F11^{-1} with hodbf_invert (Alg. 4) and uploads F12 / F21."""

    def __init__(self, fronts, N: int, eps: float = 1e-10, rank_max: int = 64, dense_max: int = 0, device: int = 0):
        L = _lib()
        for name, args in (("bf_mf_create", [C.c_int, C.c_int64, C.c_int32, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
                           ("bf_mf_destroy", [C.c_void_p]),
                           ("bf_mf_workspace_size", [C.c_void_p, C.c_int64, C.POINTER(C.c_size_t)]),
                           ("bf_mf_solve", [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                            C.c_void_p, C.c_size_t, C.c_void_p])):
            getattr(L, name).restype = C.c_int
            getattr(L, name).argtypes = args
        self.N, self.device = N, device
        self.inv, self.bfs, keep = [], [], []
        arr = (bf_front * len(fronts))()
        code = _np_dtype_code(fronts[0].F11.dtype)
        for k, f in enumerate(fronts):
            inv = HODBFInverse(f.F11, eps=eps, rank_max=rank_max, dense_max=dense_max, device=device)
            self.inv.append(inv)
            a = arr[k]
            a.parent, a.s_off, a.s_len = f.parent, f.s_off, f.s_len
            u = np.ascontiguousarray(f.u_idx, dtype=np.int64)
            keep.append(u)
            a.u_len = len(u)
            a.u_idx = u.ctypes.data_as(C.POINTER(C.c_int64)) if len(u) else None
            a.F11inv = inv.h
            if len(u):
                h12, h21 = BFHandle(f.F12, device), BFHandle(f.F21, device)
                self.bfs += [h12, h21]
                a.F12, a.F21 = h12.h, h21.h
        h = C.c_void_p()
        _check("bf_mf_create", L.bf_mf_create(code, N, len(fronts), C.cast(arr, C.c_void_p), device, C.byref(h)))
        self.h, self.code = h, code

    def close(self):
        if getattr(self, "h", None):
            _lib().bf_mf_destroy(self.h)
            self.h = None

    __del__ = close

    def workspace_size(self, nrhs: int) -> int:
        s = C.c_size_t()
        _check("bf_mf_workspace_size", _lib().bf_mf_workspace_size(self.h, nrhs, C.byref(s)))
        return s.value

    def solve(self, B: torch.Tensor, out: Optional[torch.Tensor] = None, work: Optional[torch.Tensor] = None):
        """X = M^{-1} B; B (nrhs, N) on the device."""
        assert B.is_cuda and B.dim() == 2 and B.shape[1] == self.N and B.stride(1) == 1
        nrhs = B.shape[0]
        if out is None:
            out = torch.empty_like(B)
        if work is None:
            work = torch.empty(max(self.workspace_size(nrhs), 1), dtype=torch.uint8, device=B.device)
        st = torch.cuda.current_stream()
        _check("bf_mf_solve", _lib().bf_mf_solve(self.h, nrhs, C.c_void_p(B.data_ptr()), max(B.stride(0), self.N, 1),
                                                 C.c_void_p(out.data_ptr()), max(out.stride(0), self.N, 1),
                                                 C.c_void_p(work.data_ptr()), work.numel(),
                                                 C.c_void_p(st.cuda_stream)))
        return out
