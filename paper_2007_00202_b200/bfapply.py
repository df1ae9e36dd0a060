"""Thin ctypes binding of libbfapply (include/bfapply.h).

Argument marshalling only: every step of the apply runs in the CUDA kernels of
libbfapply.so.  PyTorch provides device memory, streams and (for the distributed
apply) the NCCL process group.  There is no CPU path: if the library or a CUDA device
is missing, every call raises.

Layout: right-hand sides are torch tensors of shape (nrhs, rows), row stride `ld`
(>= rows), unit column stride -- exactly the column-major (rows x nrhs, ld) block of
the C-ABI.  Factor inputs come from ``bfinputs`` containers (packed canonical order,
the same layout the C-ABI documents).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# BF_LIB: an alternative build of the same library (A/B measurements of compile-time variants)
LIB_PATH = os.environ.get("BF_LIB") or os.path.join(_PKG, "libbfapply.so")

BF_C64, BF_C128 = 1, 2
BF_CREATE_FUSED_ONLY = 1  # bf_desc.flags (include/bfapply.h)
OPS = {"N": 0, "T": 1, "C": 2}
STATUS = {0: "BF_OK", -1: "BF_ERR_ARG", -2: "BF_ERR_SHAPE", -3: "BF_ERR_RANK", -4: "BF_ERR_PERM",
          -5: "BF_ERR_CUDA", -6: "BF_ERR_OOM", -7: "BF_ERR_NCCL", -8: "BF_ERR_DEVICE"}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class bf_desc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("L", C.c_int32), ("lc", C.c_int32), ("flags", C.c_int32),
                ("m", C.c_int64), ("n", C.c_int64),
                ("row_leaf_ptr", _i64p), ("col_leaf_ptr", _i64p),
                ("row_perm", _i64p), ("col_perm", _i64p),
                ("rank_row", _i32p), ("rank_col", _i32p),
                ("U", C.c_void_p), ("R", C.c_void_p), ("B", C.c_void_p), ("W", C.c_void_p),
                ("Vt", C.c_void_p),
                ("len_U", C.c_int64), ("len_R", C.c_int64), ("len_B", C.c_int64),
                ("len_W", C.c_int64), ("len_Vt", C.c_int64),
                ("level_maps", C.POINTER(_i32p))]


class hodbf_desc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("LH", C.c_int32), ("n", C.c_int64),
                ("leaf_ptr", _i64p), ("perm", _i64p), ("D", C.c_void_p), ("len_D", C.c_int64),
                ("offdiag", C.POINTER(bf_desc))]


class bf_info_t(C.Structure):
    _fields_ = [("factor_entries", C.c_int64), ("device_bytes", C.c_int64),
                ("launches_n", C.c_int32), ("launches_c", C.c_int32),
                ("rows_in", C.c_int64), ("rows_out", C.c_int64)]


class bf_round_info_t(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("ntasks", C.c_int32), ("factor_entries", C.c_int64),
                ("user_rows_in", C.c_int64), ("user_rows_out", C.c_int64),
                ("slab_rows_in", C.c_int64), ("slab_rows_out", C.c_int64), ("name", C.c_char * 48)]


class BFError(RuntimeError):
    def __init__(self, fn, code, msg):
        super().__init__(f"{fn}: {STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None

# (name, restype, argtypes)
_SIGS = [
    ("bf_create", C.c_int, [C.POINTER(bf_desc), C.c_int, C.POINTER(C.c_void_p)]),
    ("bf_destroy", C.c_int, [C.c_void_p]),
    ("bf_info", C.c_int, [C.c_void_p, C.POINTER(bf_info_t)]),
    ("bf_workspace_size", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_size_t)]),
    ("bf_apply", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                           C.c_void_p, C.c_size_t, C.c_void_p]),
    ("bf_apply_adj", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                               C.c_void_p, C.c_size_t, C.c_void_p]),
    ("bf_apply_op", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                              C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("bf_workspace_size_host", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_size_t)]),
    ("bf_apply_host", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("hodbf_create", C.c_int, [C.POINTER(hodbf_desc), C.c_int, C.POINTER(C.c_void_p)]),
    ("hodbf_destroy", C.c_int, [C.c_void_p]),
    ("hodbf_info", C.c_int, [C.c_void_p, C.POINTER(bf_info_t)]),
    ("hodbf_workspace_size", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_size_t)]),
    ("hodbf_apply", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                              C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("hodbf_workspace_size_host", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_size_t)]),
    ("hodbf_apply_host", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("bf_dist_create", C.c_int, [C.POINTER(bf_desc), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("bf_dist_layout", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), _i64p, _i64p]),
    ("bf_dist_local_rows", C.c_int, [C.c_void_p, C.c_int, _i64p, _i64p, _i64p, _i64p]),
    ("bf_dist_apply_pre", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_size_t, C.c_void_p]),
    ("bf_dist_apply_post", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_size_t, C.c_void_p]),
    ("bf_extract", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                             C.c_void_p]),
    ("hodbf_extract", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                C.c_void_p]),
    ("bf_accumulate", C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                C.c_void_p]),
    ("bf_rounds", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int32)]),
    ("bf_round_info", C.c_int, [C.c_void_p, C.c_int, C.c_int32, C.POINTER(bf_round_info_t)]),
    ("bf_apply_op_events", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p,
                                     C.POINTER(C.c_void_p), C.c_int32]),
    ("hodbf_rounds", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int32)]),
    ("hodbf_round_info", C.c_int, [C.c_void_p, C.c_int, C.c_int32, C.POINTER(bf_round_info_t)]),
    ("hodbf_apply_events", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p,
                                     C.POINTER(C.c_void_p), C.c_int32]),
    ("bf_status_string", C.c_char_p, [C.c_int]),
    ("bf_last_error", C.c_char_p, []),
    ("bf_version", C.c_char_p, []),
]


def lib():
    """Load libbfapply.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                               " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(fn, code):
    if code != 0:
        raise BFError(fn, code, lib().bf_last_error().decode())


def _np_dtype_code(dt) -> int:
    dt = np.dtype(dt)
    if dt == np.complex128:
        return BF_C128
    if dt == np.complex64:
        return BF_C64
    raise TypeError(f"unsupported dtype {dt}")


def _torch_dtype(code):
    return torch.complex128 if code == BF_C128 else torch.complex64


def _ptr(a: Optional[np.ndarray], ctype=None):
    if a is None:
        return None
    if ctype is None:
        return C.c_void_p(a.ctypes.data) if a.size else None
    return a.ctypes.data_as(C.POINTER(ctype))


class _Keep:
    """Holds the numpy arrays a descriptor points into until create returns."""

    def __init__(self):
        self.arrs = []

    def __call__(self, a, dtype=None):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.arrs.append(a)
        return a


def make_desc(bf, keep: _Keep, tree_local: bool = False, level_maps=None) -> bf_desc:
    """bf_desc for a bfinputs.Butterfly (packed arrays are passed straight through).

    ``level_maps``: optional list of L + 1 entries (None or a 2^L int array: storage slot ->
    canonical block index of that level); the stages of ``bf`` are then in slot order
    (include/bfapply.h, bf_desc.level_maps)."""
    code = _np_dtype_code(bf.dtype)
    d = bf_desc()
    d.dtype, d.L, d.lc, d.m, d.n = code, bf.L, bf.lc, bf.m, bf.n
    d.row_leaf_ptr = _ptr(keep(bf.row_leaf_ptr, np.int64), C.c_int64)
    d.col_leaf_ptr = _ptr(keep(bf.col_leaf_ptr, np.int64), C.c_int64)
    if tree_local:
        d.row_perm = None
        d.col_perm = None
    else:
        d.row_perm = _ptr(keep(bf.row_perm, np.int64), C.c_int64)
        d.col_perm = _ptr(keep(bf.col_perm, np.int64), C.c_int64)
    d.rank_row = _ptr(keep(bf.rank_row(), np.int32), C.c_int32)
    d.rank_col = _ptr(keep(bf.rank_col(), np.int32), C.c_int32)
    cdt = np.complex128 if code == BF_C128 else np.complex64
    U = keep(bf.U.data, cdt)
    Rr = keep(np.concatenate([s.data for s in bf.R]) if bf.R else np.zeros(0), cdt)
    Bb = keep(bf.B.data, cdt)
    Ww = keep(np.concatenate([s.data for s in bf.W]) if bf.W else np.zeros(0), cdt)
    Vt = keep(bf.Vt.data, cdt)
    d.U, d.R, d.B, d.W, d.Vt = _ptr(U), _ptr(Rr), _ptr(Bb), _ptr(Ww), _ptr(Vt)
    d.len_U, d.len_R, d.len_B, d.len_W, d.len_Vt = U.size, Rr.size, Bb.size, Ww.size, Vt.size
    if level_maps is not None:
        if len(level_maps) != bf.L + 1:
            raise ValueError(f"level_maps needs L + 1 = {bf.L + 1} entries")
        arr = (_i32p * (bf.L + 1))()
        for l, mp in enumerate(level_maps):
            arr[l] = None if mp is None else _ptr(keep(mp, np.int32), C.c_int32)
        keep.arrs.append(arr)
        d.level_maps = C.cast(arr, C.POINTER(_i32p))
    return d


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _check_rhs(X: torch.Tensor, rows: int, code: int, name: str):
    if not X.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if X.dtype != _torch_dtype(code):
        raise TypeError(f"{name} dtype {X.dtype} != handle dtype {_torch_dtype(code)}")
    if X.dim() != 2 or X.shape[1] != rows or X.stride(1) != 1:
        raise ValueError(f"{name} must be (nrhs, {rows}) with unit column stride, got {tuple(X.shape)} {X.stride()}")
    return max(X.stride(0), rows, 1) if X.shape[0] > 1 else max(rows, 1)


class Workspace:
    """Cached device byte buffers, one per stream, grown on demand.

    Applies on different streams that do not pass an explicit ``work=`` therefore never share a
    slab buffer (the header allows concurrent applies only with distinct workspaces).  A buffer
    that is replaced by a larger one is retired with ``record_stream`` on the stream that used
    it, so the caching allocator cannot hand it out again before that stream's work on it ends.
    """

    def __init__(self, device):
        self.device = device
        self.bufs = {}

    def get(self, nbytes: int, stream=None) -> torch.Tensor:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        key = st.cuda_stream
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                buf.record_stream(st)
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self.bufs[key] = buf
        return buf


class BFHandle:
    """A butterfly uploaded to one device (bf_create)."""

    def __init__(self, bf, device: int = 0, level_maps=None, fused_only: bool = False):
        keep = _Keep()
        d = make_desc(bf, keep, level_maps=level_maps)
        d.flags = BF_CREATE_FUSED_ONLY if fused_only else 0
        h = C.c_void_p()
        _check("bf_create", lib().bf_create(C.byref(d), device, C.byref(h)))
        self.h, self.device, self.code = h, device, d.dtype
        self.m, self.n = bf.m, bf.n
        self.ws = Workspace(torch.device("cuda", device))
        inf = bf_info_t()
        _check("bf_info", lib().bf_info(h, C.byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in bf_info_t._fields_}

    @classmethod
    def from_raw(cls, h, device: int, code: int, m: int, n: int) -> "BFHandle":
        """Wrap a handle the library created (e.g. bf_random_matvec's result)."""
        self = cls.__new__(cls)
        self.h, self.device, self.code = h, device, code
        self.m, self.n = m, n
        self.ws = Workspace(torch.device("cuda", device))
        inf = bf_info_t()
        _check("bf_info", lib().bf_info(h, C.byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in bf_info_t._fields_}
        return self

    def close(self):
        if getattr(self, "h", None):
            lib().bf_destroy(self.h)
            self.h = None

    __del__ = close

    def workspace_size(self, nrhs: int) -> int:
        s = C.c_size_t()
        _check("bf_workspace_size", lib().bf_workspace_size(self.h, nrhs, C.byref(s)))
        return s.value

    def extract(self, rows, cols, stream=None) -> torch.Tensor:
        """K(rows, cols) as an (len(rows), len(cols)) device tensor (bf_extract: the sub-matrix
        as a partial matvec over the touched blocks; synchronous).  rows / cols: user indices."""
        r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
        out = torch.zeros((len(c), len(r)), dtype=_torch_dtype(self.code), device=torch.device("cuda", self.device))
        _check("bf_extract", lib().bf_extract(self.h, len(r), r.ctypes.data_as(C.c_void_p), len(c),
                                              c.ctypes.data_as(C.c_void_p), C.c_void_p(out.data_ptr()),
                                              max(len(r), 1), _stream_handle(stream)))
        return out.T

    def extract_list(self, pairs, stream=None):
        """[K(rows_k, cols_k) for (rows_k, cols_k) in pairs] (bf_extract_list: Alg. 3's list form,
        one batched evaluation; synchronous).  Each result an (len(rows_k), len(cols_k)) tensor."""
        L = lib()
        if not getattr(L, "_xl_sig", False):
            L.bf_extract_list.restype = C.c_int
            L.bf_extract_list.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_int64), C.c_void_p]
            L._xl_sig = True
        keep, outs = [], []
        n = len(pairs)
        nI, nJ, ldo = (C.c_int64 * max(n, 1))(), (C.c_int64 * max(n, 1))(), (C.c_int64 * max(n, 1))()
        rp, cp, op = (C.c_void_p * max(n, 1))(), (C.c_void_p * max(n, 1))(), (C.c_void_p * max(n, 1))()
        for k, (r, c) in enumerate(pairs):
            r = np.ascontiguousarray(np.asarray(r, dtype=np.int64))
            c = np.ascontiguousarray(np.asarray(c, dtype=np.int64))
            keep += [r, c]
            o = torch.zeros((len(c), len(r)), dtype=_torch_dtype(self.code), device=torch.device("cuda", self.device))
            outs.append(o)
            nI[k], nJ[k], ldo[k] = len(r), len(c), max(len(r), 1)
            rp[k], cp[k], op[k] = r.ctypes.data, c.ctypes.data, o.data_ptr()
        _check("bf_extract_list", L.bf_extract_list(self.h, n, nI, rp, nJ, cp, op, ldo, _stream_handle(stream)))
        return [o.T for o in outs]

    def apply(self, X: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None,
              work: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Y = K X (op N), K^H X (op C) or K^T X (op T); X, Y shaped (nrhs, rows)."""
        rin, rout = (self.n, self.m) if op == "N" else (self.m, self.n)
        ldx = _check_rhs(X, rin, self.code, "X")
        nrhs = X.shape[0]
        if out is None:
            out = torch.empty((nrhs, rout), dtype=X.dtype, device=X.device)
        ldy = _check_rhs(out, rout, self.code, "Y")
        wb = self.workspace_size(nrhs)
        if work is None:
            work = self.ws.get(wb, stream)
        _check("bf_apply_op", lib().bf_apply_op(self.h, OPS[op], nrhs, C.c_void_p(X.data_ptr()), ldx,
                                                C.c_void_p(out.data_ptr()), ldy,
                                                C.c_void_p(work.data_ptr()), work.numel(),
                                                _stream_handle(stream)))
        return out

    def rounds(self, op: str = "N"):
        """Per-launch descriptions (bf_round_info) of one apply."""
        return _rounds(lib().bf_rounds, lib().bf_round_info, self.h, op)

    def apply_events(self, X, events, op: str = "N", out=None, work=None, stream=None):
        """apply() that records events[i] before launch i and events[-1] after the last."""
        rin, rout = (self.n, self.m) if op == "N" else (self.m, self.n)
        ldx = _check_rhs(X, rin, self.code, "X")
        nrhs = X.shape[0]
        if out is None:
            out = torch.empty((nrhs, rout), dtype=X.dtype, device=X.device)
        ldy = _check_rhs(out, rout, self.code, "Y")
        if work is None:
            work = self.ws.get(self.workspace_size(nrhs), stream)
        evs = (C.c_void_p * len(events))(*[C.c_void_p(e.cuda_event) for e in events])
        _check("bf_apply_op_events", lib().bf_apply_op_events(
            self.h, OPS[op], nrhs, C.c_void_p(X.data_ptr()), ldx, C.c_void_p(out.data_ptr()), ldy,
            C.c_void_p(work.data_ptr()), work.numel(), _stream_handle(stream), evs, len(events)))
        return out

    def graph(self, X: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None,
              work: Optional[torch.Tensor] = None) -> "ApplyGraph":
        """Capture one apply on the static buffers X / out / work into a CUDA graph (the whole
        launch sequence replays with one host call: for small, launch-bound butterflies).
        Refill X in place and call .replay(); the result lands in .out."""
        return ApplyGraph(self, X, op, out, work)

    def workspace_size_host(self, nrhs: int, op: str = "N") -> int:
        s = C.c_size_t()
        _check("bf_workspace_size_host", lib().bf_workspace_size_host(self.h, OPS[op], nrhs, C.byref(s)))
        return s.value

    def apply_host(self, Xh: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None,
                   work: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """End-to-end form: X and Y in (pinned) host memory; copies inside the call, pipelined
        across calls (include/bfapply.h).  `out` is complete once `stream` synchronises."""
        rin, rout = (self.n, self.m) if op == "N" else (self.m, self.n)
        assert not Xh.is_cuda and Xh.dim() == 2 and Xh.shape[1] == rin and Xh.is_contiguous()
        nrhs = Xh.shape[0]
        if out is None:
            out = torch.empty((nrhs, rout), dtype=Xh.dtype, pin_memory=True)
        s = C.c_size_t()
        _check("bf_workspace_size_host", lib().bf_workspace_size_host(self.h, OPS[op], nrhs, C.byref(s)))
        if work is None:
            work = self.ws.get(s.value, stream)
        _check("bf_apply_host", lib().bf_apply_host(self.h, OPS[op], nrhs, C.c_void_p(Xh.data_ptr()),
                                                    max(rin, 1), C.c_void_p(out.data_ptr()), max(rout, 1),
                                                    C.c_void_p(work.data_ptr()), work.numel(),
                                                    _stream_handle(stream)))
        return out


def _rounds(fn_count, fn_info, h, op):
    n = C.c_int32()
    _check("rounds", fn_count(h, OPS[op], C.byref(n)))
    out = []
    for i in range(n.value):
        r = bf_round_info_t()
        _check("round_info", fn_info(h, OPS[op], i, C.byref(r)))
        out.append({"kernel": r.kernel, "ntasks": r.ntasks, "factor_entries": r.factor_entries,
                    "user_rows_in": r.user_rows_in, "user_rows_out": r.user_rows_out,
                    "slab_rows_in": r.slab_rows_in, "slab_rows_out": r.slab_rows_out,
                    "name": r.name.decode()})
    return out


def make_hodbf_desc(H, keep: _Keep, level_maps=None) -> hodbf_desc:
    """hodbf_desc of a bfinputs.HODBF.  ``level_maps``: optional {(l, tau): maps} for off-diagonal
    butterflies given in slot order (bf_desc.level_maps; H.offdiag[l-1][tau] then holds the
    slot-ordered butterfly)."""
    code = _np_dtype_code(H.dtype)
    cdt = np.complex128 if code == BF_C128 else np.complex64
    d = hodbf_desc()
    d.dtype, d.LH, d.n = code, H.LH, H.n
    d.leaf_ptr = _ptr(keep(H.leaf_ptr, np.int64), C.c_int64)
    d.perm = _ptr(keep(H.perm, np.int64), C.c_int64)
    D = keep(H.D.data, cdt)
    d.D, d.len_D = _ptr(D), D.size
    nbf = sum(len(lev) for lev in H.offdiag)
    arr = (bf_desc * max(nbf, 1))()
    k = 0
    for l, lev in enumerate(H.offdiag, start=1):
        for tau, b in enumerate(lev):
            maps = (level_maps or {}).get((l, tau))
            arr[k] = make_desc(b, keep, tree_local=True, level_maps=maps)
            k += 1
    keep.arrs.append(arr)
    d.offdiag = C.cast(arr, C.POINTER(bf_desc))
    return d


class ApplyGraph:
    """One butterfly / HOD-BF apply captured into a torch.cuda.CUDAGraph (see BFHandle.graph)."""

    def __init__(self, h, X: torch.Tensor, op: str, out: Optional[torch.Tensor], work: Optional[torch.Tensor]):
        nrhs = X.shape[0]
        rows_out = (h.m if op == "N" else h.n) if hasattr(h, "m") else h.n
        self.X = X
        self.out = out if out is not None else torch.empty((nrhs, rows_out), dtype=X.dtype, device=X.device)
        self.work = work if work is not None else torch.empty(max(h.workspace_size(nrhs), 1), dtype=torch.uint8,
                                                             device=X.device)
        s = torch.cuda.Stream(device=X.device)
        s.wait_stream(torch.cuda.current_stream(X.device))
        with torch.cuda.stream(s):  # warm-up outside the capture (one-time kernel attributes)
            h.apply(self.X, op, out=self.out, work=self.work, stream=s)
        torch.cuda.current_stream(X.device).wait_stream(s)
        self.g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g):
            h.apply(self.X, op, out=self.out, work=self.work, stream=torch.cuda.current_stream(X.device))

    def replay(self) -> torch.Tensor:
        self.g.replay()
        return self.out


class HODBFHandle:
    """An HOD-BF matrix uploaded to one device (hodbf_create)."""

    def __init__(self, H, device: int = 0, level_maps=None):
        keep = _Keep()
        d = make_hodbf_desc(H, keep, level_maps)
        h = C.c_void_p()
        _check("hodbf_create", lib().hodbf_create(C.byref(d), device, C.byref(h)))
        self.h, self.device, self.code, self.n = h, device, d.dtype, H.n
        self.ws = Workspace(torch.device("cuda", device))
        inf = bf_info_t()
        _check("hodbf_info", lib().hodbf_info(h, C.byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in bf_info_t._fields_}

    def close(self):
        if getattr(self, "h", None):
            lib().hodbf_destroy(self.h)
            self.h = None

    __del__ = close

    def workspace_size(self, nrhs: int) -> int:
        s = C.c_size_t()
        _check("hodbf_workspace_size", lib().hodbf_workspace_size(self.h, nrhs, C.byref(s)))
        return s.value

    def extract(self, rows, cols, stream=None) -> torch.Tensor:
        """A(rows, cols) as an (len(rows), len(cols)) device tensor (hodbf_extract; synchronous)."""
        r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
        out = torch.zeros((len(c), len(r)), dtype=_torch_dtype(self.code), device=torch.device("cuda", self.device))
        _check("hodbf_extract", lib().hodbf_extract(self.h, len(r), r.ctypes.data_as(C.c_void_p), len(c),
                                                    c.ctypes.data_as(C.c_void_p), C.c_void_p(out.data_ptr()),
                                                    max(len(r), 1), _stream_handle(stream)))
        return out.T

    def apply(self, X: torch.Tensor, op: str = "N", out=None, work=None, stream=None) -> torch.Tensor:
        ldx = _check_rhs(X, self.n, self.code, "X")
        nrhs = X.shape[0]
        if out is None:
            out = torch.empty((nrhs, self.n), dtype=X.dtype, device=X.device)
        ldy = _check_rhs(out, self.n, self.code, "Y")
        if work is None:
            work = self.ws.get(self.workspace_size(nrhs), stream)
        _check("hodbf_apply", lib().hodbf_apply(self.h, OPS[op], nrhs, C.c_void_p(X.data_ptr()), ldx,
                                                C.c_void_p(out.data_ptr()), ldy,
                                                C.c_void_p(work.data_ptr()), work.numel(),
                                                _stream_handle(stream)))
        return out

    def rounds(self, op: str = "N"):
        return _rounds(lib().hodbf_rounds, lib().hodbf_round_info, self.h, op)

    def graph(self, X: torch.Tensor, op: str = "N", out=None, work=None) -> ApplyGraph:
        """See BFHandle.graph."""
        return ApplyGraph(self, X, op, out, work)

    def apply_events(self, X, events, op: str = "N", out=None, work=None, stream=None):
        ldx = _check_rhs(X, self.n, self.code, "X")
        nrhs = X.shape[0]
        if out is None:
            out = torch.empty((nrhs, self.n), dtype=X.dtype, device=X.device)
        ldy = _check_rhs(out, self.n, self.code, "Y")
        if work is None:
            work = self.ws.get(self.workspace_size(nrhs), stream)
        evs = (C.c_void_p * len(events))(*[C.c_void_p(e.cuda_event) for e in events])
        _check("hodbf_apply_events", lib().hodbf_apply_events(
            self.h, OPS[op], nrhs, C.c_void_p(X.data_ptr()), ldx, C.c_void_p(out.data_ptr()), ldy,
            C.c_void_p(work.data_ptr()), work.numel(), _stream_handle(stream), evs, len(events)))
        return out

    def apply_host(self, Xh: torch.Tensor, op: str = "N", out=None, work=None, stream=None):
        assert not Xh.is_cuda and Xh.dim() == 2 and Xh.shape[1] == self.n and Xh.is_contiguous()
        nrhs = Xh.shape[0]
        if out is None:
            out = torch.empty((nrhs, self.n), dtype=Xh.dtype, pin_memory=True)
        s = C.c_size_t()
        _check("hodbf_workspace_size_host", lib().hodbf_workspace_size_host(self.h, nrhs, C.byref(s)))
        if work is None:
            work = self.ws.get(s.value, stream)
        _check("hodbf_apply_host", lib().hodbf_apply_host(self.h, OPS[op], nrhs, C.c_void_p(Xh.data_ptr()),
                                                          max(self.n, 1), C.c_void_p(out.data_ptr()),
                                                          max(self.n, 1), C.c_void_p(work.data_ptr()),
                                                          work.numel(), _stream_handle(stream)))
        return out


# ---- C-ABI-named convenience functions (same names as include/bfapply.h) ------------
def bf_create(bf, device: int = 0) -> BFHandle:
    return BFHandle(bf, device)


def bf_apply(h: BFHandle, X, **kw):
    return h.apply(X, "N", **kw)


def bf_apply_adj(h: BFHandle, X, **kw):
    return h.apply(X, "C", **kw)


def bf_apply_op(h: BFHandle, op: str, X, **kw):
    return h.apply(X, op, **kw)


def hodbf_create(H, device: int = 0) -> HODBFHandle:
    return HODBFHandle(H, device)


def hodbf_apply(h: HODBFHandle, X, op: str = "N", **kw):
    return h.apply(X, op, **kw)


def version() -> str:
    return lib().bf_version().decode()
