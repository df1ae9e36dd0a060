"""Multi-process (gloo, world 2 and 4) CPU test of the tree-partitioned HOD-BF's exchange
(dist.TreeHODBF): every rank builds HOST-ONLY plans of the butterflies at the
distributed levels, tags every element of its column sides' send regions with (level,
butterfly node, centre block, element), runs the same grouped send / receive the GPU path uses
(batch_isend_irecv over gloo instead of NCCL) and checks that every received slab carries the
tag its row side's map expects, and that it came from the sibling node's ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sizes(bf, op):
    """Rows of every centre block's slab, canonical (tau, nu) order: r^lc (op N), c^lc (op C)."""
    L, lc = bf.L, bf.lc
    return bf.rank_row()[: 1 << L] if op == "N" else bf.rank_col()[lc << L:]


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from bfinputs.configs import helmholtz_plane_hodbf
        from paper_2007_00202_b200.dist import TreeHODBF
        H = helmholtz_plane_hodbf(16, 16, 10.0, 1e-4)
        t = TreeHODBF(H, rank, world, device=None)
        p = world.bit_length() - 1
        lo, hi = t.rows()
        assert (lo, hi) == H.node_range(p, rank)
        nrhs = 3
        for op in ("N", "C"):
            bufs = t.buffers(op, nrhs)
            for lev, pl, (sv, rv) in zip(t.levels, t.exchange_plan(op, nrhs), bufs):
                l = lev["l"]
                a = rank >> (p - l)
                b = a ^ 1
                assert [peer for peer, _ in sv] == [(b << (p - l)) + k for k in range(1 << (p - l))]
                Hc, Hr = pl["Hc"], pl["Hr"]
                node_c = b if op == "N" else a   # butterfly whose column side runs here
                node_r = a if op == "N" else b   # butterfly whose row side runs here
                sblk, _ = Hc.exchange_blocks(op)
                _, rblk = Hr.exchange_blocks(op)
                size_c = _sizes(H.offdiag[l - 1][node_c], op)
                size_r = _sizes(H.offdiag[l - 1][node_r], op)
                send = torch.cat([v for _, v in sv]).view(-1, 2) if sv else torch.zeros(0, 2)
                assert send.shape[0] == int(sum(size_c[sblk])) * nrhs
                k = 0
                for blk in sblk:
                    for e in range(int(size_c[blk]) * nrhs):
                        send[k, 0] = 1000.0 * l + node_c
                        send[k, 1] = 100000.0 * blk + e
                        k += 1
                # write the tags back into the per-peer views
                at = 0
                for _, v in sv:
                    n = v.numel() // 2
                    v.view(-1, 2).copy_(send[at:at + n])
                    at += n
            t.exchange(op, nrhs)
            for lev, pl, (sv, rv) in zip(t.levels, t.exchange_plan(op, nrhs), t.buffers(op, nrhs)):
                l = lev["l"]
                a = rank >> (p - l)
                node_r = a if op == "N" else a ^ 1
                _, rblk = pl["Hr"].exchange_blocks(op)
                size_r = _sizes(H.offdiag[l - 1][node_r], op)
                recv = torch.cat([v for _, v in rv]).view(-1, 2)
                assert recv.shape[0] == int(sum(size_r[rblk])) * nrhs
                k = 0
                for blk in rblk:
                    for e in range(int(size_r[blk]) * nrhs):
                        assert recv[k, 0] == 1000.0 * l + node_r and recv[k, 1] == 100000.0 * blk + e, (op, l, blk, e)
                        k += 1
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException:  # report, do not hang the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4])
def test_tree_hodbf_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]
