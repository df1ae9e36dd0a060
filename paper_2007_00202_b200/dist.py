"""Distributed butterfly apply: one process per GPU (BASELINE north_star).

P = 2^p ranks.  Rank g owns the column subtree nu_g at level p of T_S (its V leaves, W
stages and the centre products B for nu under nu_g) and the row subtree tau_g at level p of
T_O (its R stages and U leaves).  One apply is

    bf_dist_apply_pre   (libbfapply kernels: leaf V, W stages, centre B -> send region)
    all-to-all          (NCCL over NVLink / NVSwitch: centre slabs nu-owner -> tau-owner)
    bf_dist_apply_post  (libbfapply kernels: R stages, leaf U -> Y_loc)

for op N; op C / T runs the mirror image (row subtree first).  The exchange is the only
data-path collective: the paper's own distributed algorithm is "omitted", so this
layout is the build's; the closure argument (z^l_{tau,nu} depends only on
X(S_nu), both contributions to y^{l+1}_{tau'} share tau = tau'>>1) is P:302-317.

This module is argument marshalling around the C-ABI plus the collective call: every
arithmetic step runs in libbfapply's kernels.  With ``device=None`` the handle is a
HOST-ONLY plan (bf_dist_create with device < 0): its layouts and exchange maps drive the
multi-process CPU (gloo) tests of the exchange logic.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from .bfapply import OPS, BFError, Workspace, _Keep, _check, _check_rhs, _stream_handle, _torch_dtype, lib, make_desc

_SIGS = [
    ("bf_dist_exchange_blocks", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("bf_dist_slab_format", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    ("bf_dist_exchange_level", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int32)]),
    ("bf_dist_apply_pre_p2p", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_size_t, C.POINTER(C.c_void_p), C.c_void_p]),
    ("bf_nccl_available", C.c_int, []),
    ("bf_nccl_get_unique_id", C.c_int, [C.c_void_p]),
    ("bf_nccl_comm_init", C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("bf_nccl_comm_destroy", C.c_int, [C.c_void_p]),
    ("bf_create_dist", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("bf_apply_dist", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                C.c_void_p, C.c_size_t, C.c_void_p]),
]


def _lib():
    L = lib()
    for name, res, args in _SIGS:
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def _opk(op: str) -> int:
    return 0 if op == "N" else 1


class NcclComm:
    """A library-owned NCCL communicator (bf_nccl_comm_init) over the ranks of ``group``: rank 0
    draws the ncclUniqueId, the process group carries its 128 bytes to the others (any backend,
    gloo included), then every rank joins on its device.  Used by DistBFHandle(comm=...), whose
    apply is then the single C-ABI call bf_apply_dist (pre, grouped ncclSend / ncclRecv, post)."""

    def __init__(self, device: int, group=None):
        L = _lib()
        if not L.bf_nccl_available():
            raise BFError("bf_nccl_available", -7, "NCCL cannot be loaded")
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_char * 128)()
        if rank == 0:
            _check("bf_nccl_get_unique_id", L.bf_nccl_get_unique_id(uid))
        if world > 1:
            obj = [bytes(uid) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            C.memmove(uid, obj[0], 128)
        c = C.c_void_p()
        _check("bf_nccl_comm_init", L.bf_nccl_comm_init(world, uid, rank, int(device), C.byref(c)))
        self.ptr, self.rank, self.world, self.device = c, rank, world, device

    def close(self):
        """Destroy the communicator (after every DistBFHandle using it: each holds a reference)."""
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            try:
                _lib().bf_nccl_comm_destroy(self.ptr)
            except Exception:  # interpreter shutdown: the library may already be gone
                pass
        self.ptr = None

    __del__ = close


class DistBFHandle:
    """This rank's share of a butterfly split over ``world`` processes (bf_dist_create; with
    ``comm`` an NcclComm, bf_create_dist: the library then runs the exchange itself)."""

    def __init__(self, bf, rank: int, world: int, device: Optional[int] = 0, group=None,
                 comm: Optional[NcclComm] = None):
        keep = _Keep()
        d = make_desc(bf, keep)
        h = C.c_void_p()
        dev = -1 if device is None else int(device)
        if comm is not None:
            _check("bf_create_dist", _lib().bf_create_dist(C.byref(d), rank, world, comm.ptr, dev, C.byref(h)))
        else:
            _check("bf_dist_create", _lib().bf_dist_create(C.byref(d), rank, world, dev, C.byref(h)))
        self.h, self.rank, self.world, self.device, self.code = h, rank, world, device, d.dtype
        self.group = group
        self.comm = comm
        self.cs = 16 if d.dtype == 2 else 8
        self.m, self.n = bf.m, bf.n
        self.ws = Workspace(torch.device("cuda", device)) if device is not None else None
        self._rows = {}
        for op in ("N", "C"):
            ri, ro, ui, uo = (C.c_int64() for _ in range(4))
            _check("bf_dist_local_rows", _lib().bf_dist_local_rows(h, OPS[op], C.byref(ri), C.byref(ro),
                                                                    C.byref(ui), C.byref(uo)))
            self._rows[op] = (ri.value, ro.value, ui.value, uo.value)
        self._rows["T"] = self._rows["C"]

    def close(self):
        if getattr(self, "h", None):
            lib().bf_destroy(self.h)
            self.h = None

    __del__ = close

    # ---- layout -------------------------------------------------------------------
    def layout(self, op: str, nrhs: int):
        """(work_bytes, send_off, recv_off, send_counts, recv_counts) -- offsets in bytes,
        counts in complex elements per peer (bf_dist_layout)."""
        wb, so, ro = C.c_size_t(), C.c_size_t(), C.c_size_t()
        sc = (C.c_int64 * self.world)()
        rc = (C.c_int64 * self.world)()
        _check("bf_dist_layout", _lib().bf_dist_layout(self.h, OPS[op], nrhs, C.byref(wb), C.byref(so), C.byref(ro),
                                                        sc, rc))
        return wb.value, so.value, ro.value, list(sc), list(rc)

    def exchange_blocks(self, op: str):
        """Centre blocks in send-region and recv-region order (bf_dist_exchange_blocks)."""
        ns, nr = C.c_int64(), C.c_int64()
        _check("bf_dist_exchange_blocks", _lib().bf_dist_exchange_blocks(self.h, OPS[op], C.byref(ns), None,
                                                                          C.byref(nr), None))
        s = np.zeros(max(ns.value, 1), dtype=np.int64)
        r = np.zeros(max(nr.value, 1), dtype=np.int64)
        _check("bf_dist_exchange_blocks", _lib().bf_dist_exchange_blocks(
            self.h, OPS[op], C.byref(ns), s.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(nr),
            r.ctypes.data_as(C.POINTER(C.c_int64))))
        return s[:ns.value], r[:nr.value]

    def exchange_level(self, op: str = "N") -> int:
        """The level whose slabs the exchange moves (bf_dist_exchange_level): lc on the generic
        split, the pass-count-minimising level on the fused one."""
        v = C.c_int32()
        _check("bf_dist_exchange_level", _lib().bf_dist_exchange_level(self.h, OPS[op], C.byref(v)))
        return v.value

    def slab_format(self) -> int:
        """0: generic block-contiguous send / recv regions; 1: fused-kernel half-slab chunks
        (include/bfapply.h, bf_dist_slab_format)."""
        f = C.c_int32()
        _check("bf_dist_slab_format", _lib().bf_dist_slab_format(self.h, C.byref(f)))
        return f.value

    def local_rows(self, op: str):
        """(rows_in, rows_out, user_off_in, user_off_out): this rank's slice of X and Y."""
        return self._rows[op]

    def local_input(self, X: np.ndarray, op: str = "N") -> np.ndarray:
        """This rank's rows of a full (rows, nrhs) right-hand-side block."""
        ri, _, ui, _ = self._rows[op]
        return X[ui:ui + ri]

    def empty_output(self, nrhs: int, op: str = "N") -> torch.Tensor:
        _, ro, _, _ = self._rows[op]
        return torch.empty((nrhs, ro), dtype=_torch_dtype(self.code), device=torch.device("cuda", self.device))

    def launches(self, op: str = "N") -> int:
        n = C.c_int32()
        _check("bf_rounds", lib().bf_rounds(self.h, OPS[op], C.byref(n)))
        return n.value

    # ---- apply --------------------------------------------------------------------
    def exchange(self, work: torch.Tensor, op: str, nrhs: int):
        """The all-to-all of the centre slabs inside `work` (send region -> recv region)."""
        _, so, ro, sc, rc = self.layout(op, nrhs)
        rdt = torch.float64 if self.cs == 16 else torch.float32  # NCCL moves the (re, im) pairs
        send = work[so:so + sum(sc) * self.cs].view(rdt)
        recv = work[ro:ro + sum(rc) * self.cs].view(rdt)
        if self.world == 1:
            recv.copy_(send)
            return
        dist.all_to_all_single(recv, send, output_split_sizes=[2 * c for c in rc],
                               input_split_sizes=[2 * c for c in sc], group=self.group)

    def enable_p2p(self, nrhs: int, op: str = "N"):
        """Fused peer-memory exchange (bf_dist_apply_pre_p2p): the workspace becomes a torch
        symmetric-memory buffer mapped on every rank, so the pass that ends at the centre stores
        its slabs straight into the receivers' recv regions over NVLink; a device-side barrier
        replaces the all-to-all.  Needs the fused split (slab_format() == 1)."""
        import torch.distributed._symmetric_memory as symm_mem
        assert self.slab_format() == 1, "peer-memory exchange needs the fused split"
        wb, so, ro, sc, rc = self.layout(op, nrhs)
        buf = symm_mem.empty(wb, dtype=torch.uint8, device=torch.device("cuda", self.device))
        grp = self.group if self.group is not None else dist.group.WORLD
        hdl = symm_mem.rendezvous(buf, grp)
        self._p2p = {"key": (op, nrhs), "work": buf, "hdl": hdl,
                     "peers": (C.c_void_p * self.world)(*[int(pt) + ro for pt in hdl.buffer_ptrs])}

    def apply(self, Xloc: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None,
              work: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Y_loc = (K X)_loc (op N) or (K^H X)_loc (op C) / (K^T X)_loc (op T)."""
        p2p = getattr(self, "_p2p", None)
        if p2p is not None and p2p["key"] == (op, Xloc.shape[0]):
            return self._apply_p2p(Xloc, op, out, stream)
        if self.ws is None:
            raise BFError("bf_dist_apply_pre", -8, "host-only plan cannot apply")
        ri, ro, _, _ = self._rows[op]
        ldx = _check_rhs(Xloc, ri, self.code, "X_loc")
        nrhs = Xloc.shape[0]
        if out is None:
            out = self.empty_output(nrhs, op)
        ldy = _check_rhs(out, ro, self.code, "Y_loc")
        wb = self.layout(op, nrhs)[0]
        if work is None:
            work = self.ws.get(wb, stream)
        st = _stream_handle(stream)
        if self.comm is not None:  # library-owned NCCL: one C-ABI call, exchange included
            _check("bf_apply_dist", _lib().bf_apply_dist(self.h, OPS[op], nrhs, C.c_void_p(Xloc.data_ptr()), ldx,
                                                         C.c_void_p(out.data_ptr()), ldy, C.c_void_p(work.data_ptr()),
                                                         work.numel(), st))
            return out
        _check("bf_dist_apply_pre", lib().bf_dist_apply_pre(self.h, OPS[op], nrhs, C.c_void_p(Xloc.data_ptr()), ldx,
                                                             C.c_void_p(work.data_ptr()), work.numel(), st))
        # NCCL orders the all-to-all against torch's current stream: make that the apply's stream,
        # so the collective reads the send region after pre and post reads the recv region after it
        with torch.cuda.stream(self._torch_stream(stream)):
            self.exchange(work, op, nrhs)
        _check("bf_dist_apply_post", lib().bf_dist_apply_post(self.h, OPS[op], nrhs, C.c_void_p(out.data_ptr()), ldy,
                                                               C.c_void_p(work.data_ptr()), work.numel(), st))
        return out

    def _apply_p2p(self, Xloc, op, out, stream):
        p2p = self._p2p
        ri, ro, _, _ = self._rows[op]
        ldx = _check_rhs(Xloc, ri, self.code, "X_loc")
        nrhs = Xloc.shape[0]
        if out is None:
            out = self.empty_output(nrhs, op)
        ldy = _check_rhs(out, ro, self.code, "Y_loc")
        work = p2p["work"]
        st = _stream_handle(stream)
        _check("bf_dist_apply_pre_p2p", _lib().bf_dist_apply_pre_p2p(
            self.h, OPS[op], nrhs, C.c_void_p(Xloc.data_ptr()), ldx, C.c_void_p(work.data_ptr()), work.numel(),
            p2p["peers"], st))
        ts = self._torch_stream(stream)
        with torch.cuda.stream(ts):   # the symmetric-memory barriers are issued on the current stream
            p2p["hdl"].barrier(channel=0)   # every sender's slabs have landed
        _check("bf_dist_apply_post", lib().bf_dist_apply_post(self.h, OPS[op], nrhs, C.c_void_p(out.data_ptr()), ldy,
                                                               C.c_void_p(work.data_ptr()), work.numel(), st))
        with torch.cuda.stream(ts):
            p2p["hdl"].barrier(channel=0)   # every receiver has read them (the next pre may write)
        return out

    def _torch_stream(self, stream):
        return stream if stream is not None else torch.cuda.current_stream(torch.device("cuda", self.device))

    def time_e2e(self, X_loc_host: torch.Tensor, op: str, steps: int, alg_bytes: int):
        """End-to-end timing through the public API: pinned host X_loc -> device, apply,
        device -> pinned host Y_loc, every step; max over ranks of the CUDA-event time.  The copies
        are pipelined like bf_apply_host: two device / host buffer sets, H2D and D2H on their own
        streams, so step k+1's H2D and apply overlap step k's D2H (the apply and its collective stay
        on the current stream, in the same order on every rank)."""
        Xp = [X_loc_host.contiguous().pin_memory() for _ in range(2)]
        nrhs = Xp[0].shape[0]
        _, ro, _, _ = self._rows[op]
        Yp = [torch.empty((nrhs, ro), dtype=Xp[0].dtype).pin_memory() for _ in range(2)]
        Xd = [torch.empty_like(Xp[0], device=torch.device("cuda", self.device)) for _ in range(2)]
        Yd = [self.empty_output(nrhs, op) for _ in range(2)]
        cur = torch.cuda.current_stream(self.device)
        s_in, s_out = torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_cmp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def run(n):
            s_in.wait_stream(cur)
            for k in range(n):
                b = k & 1
                if k >= 2:
                    s_in.wait_event(ev_out[b])  # step k - 2's D2H (after its apply) freed set b
                with torch.cuda.stream(s_in):
                    Xd[b].copy_(Xp[b], non_blocking=True)
                    ev_in[b].record(s_in)
                cur.wait_event(ev_in[b])
                self.apply(Xd[b], op, out=Yd[b])
                ev_cmp[b].record(cur)
                s_out.wait_event(ev_cmp[b])
                with torch.cuda.stream(s_out):
                    Yp[b].copy_(Yd[b], non_blocking=True)
                    ev_out[b].record(s_out)
            cur.wait_stream(s_out)

        run(2)
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        run(steps)
        e1.record(cur)
        torch.cuda.synchronize()
        Xp, Yp = Xp[0], Yp[0]
        ms = e0.elapsed_time(e1) / steps
        if self.world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=torch.device("cuda", self.device))
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            ms = float(t.item())
            hb = torch.tensor([Xp.numel() * self.cs, Yp.numel() * self.cs], dtype=torch.int64,
                              device=torch.device("cuda", self.device))
            dist.all_reduce(hb, group=self.group)
            h2d, d2h = int(hb[0].item()), int(hb[1].item())
        else:
            h2d, d2h = Xp.numel() * self.cs, Yp.numel() * self.cs
        return {"value": alg_bytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "DistBFHandle.apply (pinned host X_loc/Y_loc per rank, copies inside the timed region, H2D / D2H pipelined with the applies on two copy streams)"}


def rhs_shard(nrhs: int, rank: int, world: int):
    """Columns [c0, c1) of an nrhs-column block owned by `rank` (contiguous, balanced)."""
    base, rem = divmod(nrhs, world)
    c0 = rank * base + min(rank, rem)
    return c0, c0 + base + (1 if rank < rem else 0)


class ShardedHODBF:
    """HOD-BF apply with the right-hand sides sharded over the ranks (the layout
    for configs 3-4, which are tensor-pipe bound).  Every rank holds the full HOD-BF on its GPU
    and applies it to its own columns; there is no data-path collective.  ``apply`` takes and
    returns the rank's (ncols_loc, n) column block; ``columns(nrhs)`` says which columns."""

    def __init__(self, H, rank: int, world: int, device: int = 0):
        from .bfapply import HODBFHandle
        self.h = HODBFHandle(H, device)
        self.rank, self.world, self.n = rank, world, H.n

    def columns(self, nrhs: int):
        return rhs_shard(nrhs, self.rank, self.world)

    def apply(self, Xloc: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None) -> torch.Tensor:
        return self.h.apply(Xloc, op, out=out)


def sub_hodbf(H, p: int, g: int):
    """The HOD-BF of T_H subtree g at level p (P:542 restricted to the rows and columns of that
    node): its 2^(LH-p) dense leaves and its butterflies at levels p+1..LH, re-indexed as levels
    1..LH-p, in tree order (identity perm)."""
    from bfinputs.factors import HODBF, Stage
    lo, hi = H.node_range(p, g)
    w = 1 << (H.LH - p)
    leaf_ptr = np.asarray(H.leaf_ptr[g * w:(g + 1) * w + 1], dtype=np.int64) - lo
    D = Stage.from_blocks([H.D.block(i) for i in range(g * w, (g + 1) * w)], H.D.data.dtype)
    off = [[H.offdiag[l - 1][t] for t in range(g << (l - p), (g + 1) << (l - p))] for l in range(p + 1, H.LH + 1)]
    return HODBF(hi - lo, H.LH - p, leaf_ptr, np.arange(hi - lo, dtype=np.int64), D, off, H.dtype)


class TreeHODBF:
    """HOD-BF apply distributed by tree node.  P = 2^p ranks; rank g owns
    the T_H node g at level p: the rows and columns of A in it (X and Y rows in HOD-BF tree
    order, positions ``rows()``).

    * The dense leaves and the sibling butterflies at levels l > p lie inside the node: a local
      HOD-BF (``sub_hodbf``) applies them, no communication.
    * A sibling pair (a, b) at level l <= p spans 2^(p-l) ranks on each side.  Its butterflies
      B_a = A(T_a, T_b) and B_b = A(T_b, T_a) run as the bf_dist split over 2^(p-l) virtual
      ranks (``DistBFHandle``), virtual rank v of a node being physical rank node * 2^(p-l) + v:
      op N runs the column side (leaf V, W stages, centre B) of B_b and the row side (R stages,
      leaf U) of B_a on the ranks of node a (op C the column side of B_a^H and the row side of
      B_b^H), so every centre slab travels from the ranks of one node to the ranks of its
      sibling.
    * All levels' centre slabs move in one grouped send / receive per apply
      (``torch.distributed.batch_isend_irecv``: NCCL over NVLink / NVSwitch, gloo on CPU); the
      row sides then write scratch blocks that ``bf_accumulate`` adds into the local result.

    Every arithmetic step runs in libbfapply's kernels; this class is marshalling.  With
    ``device=None`` only the host-side plans exist (layouts, exchange maps: the gloo tests)."""

    def __init__(self, H, rank: int, world: int, device: Optional[int] = 0, group=None):
        p = world.bit_length() - 1
        if (1 << p) != world or p > H.LH - 1:
            raise ValueError("TreeHODBF needs a power-of-two world of at most 2^(LH-1) ranks")
        from .bfapply import HODBFHandle
        self.p, self.rank, self.world, self.device, self.group = p, rank, world, device, group
        self.lo, self.hi = H.node_range(p, rank)
        self.local = HODBFHandle(sub_hodbf(H, p, rank), device) if device is not None else None
        self.levels = []
        for l in range(1, p + 1):
            a = rank >> (p - l)
            b = a ^ 1
            Pv = 1 << (p - l)
            v = rank - (a << (p - l))
            Ha = DistBFHandle(H.offdiag[l - 1][a], v, Pv, device)  # rows T_a (this rank's), cols T_b
            Hb = DistBFHandle(H.offdiag[l - 1][b], v, Pv, device)  # rows T_b, cols T_a (this rank's)
            a0 = H.node_range(l, a)[0]
            # the virtual rank's slices are this rank's node: same rows in both butterflies
            assert Ha.local_rows("N")[1] == self.hi - self.lo and Ha.local_rows("N")[3] == self.lo - a0
            assert Hb.local_rows("N")[0] == self.hi - self.lo and Hb.local_rows("N")[2] == self.lo - a0
            self.levels.append({"l": l, "Ha": Ha, "Hb": Hb, "peers": [(b << (p - l)) + q for q in range(Pv)],
                                "work": {}})
        self.code = self.levels[0]["Ha"].code if self.levels else None
        self.cs = 16 if H.dtype == np.complex128 else 8

    def rows(self):
        """[lo, hi): this rank's positions in the HOD-BF tree order (X_loc / Y_loc rows)."""
        return self.lo, self.hi

    def _sides(self, lev, op: str):
        """(column-side handle, row-side handle) of level `lev` for op."""
        return (lev["Hb"], lev["Ha"]) if op == "N" else (lev["Ha"], lev["Hb"])

    def exchange_plan(self, op: str, nrhs: int):
        """Per level: the byte ranges of the column side's send region (one per sibling-node
        peer) and of the row side's recv region, with the physical peer ranks."""
        plan = []
        for lev in self.levels:
            Hc, Hr = self._sides(lev, op)
            wbc, so, _, sc, _ = Hc.layout(op, nrhs)
            wbr, _, ro, _, rc = Hr.layout(op, nrhs)
            sends, recvs, s_at, r_at = [], [], so, ro
            for q, peer in enumerate(lev["peers"]):
                sends.append((peer, s_at, sc[q] * self.cs))
                recvs.append((peer, r_at, rc[q] * self.cs))
                s_at += sc[q] * self.cs
                r_at += rc[q] * self.cs
            plan.append({"l": lev["l"], "Hc": Hc, "Hr": Hr, "work_bytes": (wbc, wbr), "sends": sends, "recvs": recvs})
        return plan

    def _works(self, lev, op, nrhs, wbc, wbr):
        key = (op, nrhs)
        if key not in lev["work"]:
            dev = torch.device("cuda", self.device) if self.device is not None else "cpu"
            lev["work"][key] = (torch.zeros(max(wbc, 1), dtype=torch.uint8, device=dev),
                                torch.zeros(max(wbr, 1), dtype=torch.uint8, device=dev))
        return lev["work"][key]

    def pre(self, Xloc: torch.Tensor, op: str = "N", stream=None):
        """Every level's column side on this rank's X rows (send regions filled)."""
        nrhs = Xloc.shape[0]
        st = _stream_handle(stream)
        for lev, pl in zip(self.levels, self.exchange_plan(op, nrhs)):
            wc, _ = self._works(lev, op, nrhs, *pl["work_bytes"])
            Hc = pl["Hc"]
            ldx = _check_rhs(Xloc, self.hi - self.lo, self.code, "X_loc")
            _check("bf_dist_apply_pre", lib().bf_dist_apply_pre(Hc.h, OPS[op], nrhs, C.c_void_p(Xloc.data_ptr()), ldx,
                                                                 C.c_void_p(wc.data_ptr()), wc.numel(), st))

    def buffers(self, op: str, nrhs: int):
        """Per level: [(peer, send view)], [(peer, recv view)] (float views of the work buffers)."""
        rdt = torch.float64 if self.cs == 16 else torch.float32
        out = []
        for lev, pl in zip(self.levels, self.exchange_plan(op, nrhs)):
            wc, wr = self._works(lev, op, nrhs, *pl["work_bytes"])
            sv = [(peer, wc[o:o + n].view(rdt)) for peer, o, n in pl["sends"]]
            rv = [(peer, wr[o:o + n].view(rdt)) for peer, o, n in pl["recvs"]]
            out.append((sv, rv))
        return out

    def exchange(self, op: str, nrhs: int):
        """One grouped send / receive of every level's centre slabs between sibling nodes."""
        ops = []
        for sv, rv in self.buffers(op, nrhs):
            ops += [dist.P2POp(dist.isend, t, peer, group=self.group) for peer, t in sv if t.numel()]
            ops += [dist.P2POp(dist.irecv, t, peer, group=self.group) for peer, t in rv if t.numel()]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def post(self, Yloc: torch.Tensor, op: str = "N", stream=None):
        """Every level's row side from its recv region, accumulated into Y_loc (bf_accumulate)."""
        nrhs = Yloc.shape[0]
        rows = self.hi - self.lo
        ldy = _check_rhs(Yloc, rows, self.code, "Y_loc")
        st = _stream_handle(stream)
        tmp = torch.empty_like(Yloc)
        for lev, pl in zip(self.levels, self.exchange_plan(op, nrhs)):
            _, wr = self._works(lev, op, nrhs, *pl["work_bytes"])
            Hr = pl["Hr"]
            _check("bf_dist_apply_post", lib().bf_dist_apply_post(Hr.h, OPS[op], nrhs, C.c_void_p(tmp.data_ptr()), ldy,
                                                                   C.c_void_p(wr.data_ptr()), wr.numel(), st))
            _check("bf_accumulate", lib().bf_accumulate(self.code, rows, nrhs, C.c_void_p(tmp.data_ptr()), ldy,
                                                        C.c_void_p(Yloc.data_ptr()), ldy, st))

    def apply(self, Xloc: torch.Tensor, op: str = "N", out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Y_loc = (A X)_loc (op N) or (A^H X)_loc (op C) for this rank's rows (tree order)."""
        if self.local is None:
            raise BFError("hodbf_apply", -8, "host-only plan cannot apply")
        Y = self.local.apply(Xloc, op, out=out)
        self.pre(Xloc, op)
        self.exchange(op, Xloc.shape[0])  # NCCL's stream waits for the current one (the send regions)
        self.post(Y, op)
        return Y
