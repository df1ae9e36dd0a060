"""Multi-process (gloo, world size 2 and 4) CPU tests of the distributed apply's host logic:
the rank-local row ranges, the per-peer counts of the centre-slab all-to-all and the
order in which every sender packs and every receiver unpacks the slabs.

Each rank builds a HOST-ONLY plan (bf_dist_create with device < 0: nothing is uploaded),
tags every element of its send region with (centre block, row, column), runs the same
DistBFHandle.exchange() the GPU path uses -- all_to_all_single over gloo instead of
NCCL -- and checks that every received slab carries the tag the receiver's map expects.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from bfinputs import random_butterfly, random_ranks_butterfly


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _subtree_perm(n, leaf_ptr, L, p, seed):
    """A permutation under which every level-p subtree maps to a contiguous user range
    (shuffled inside each subtree, subtrees kept in order)."""
    rng = np.random.default_rng(seed)
    perm = np.empty(n, dtype=np.int64)
    w = 1 << (L - p)
    for g in range(1 << p):
        a, b = int(leaf_ptr[g * w]), int(leaf_ptr[(g + 1) * w])
        perm[a:b] = a + rng.permutation(b - a)
    return perm


def _case(kind):
    if kind == "fast":  # uniform rank 16: the fused kernels' split and exchange format
        bf = random_butterfly(L=8, leaf=16, r=16, seed=7)
    elif kind == "uniform":
        bf = random_butterfly(L=6, leaf=4, r=3, seed=5)
    else:
        rng = np.random.default_rng(3)
        bf = random_ranks_butterfly(6, rng.integers(0, 5, 64), rng.integers(1, 5, 64), seed=3, rmin=1, rmax=6)
    bf.row_perm = _subtree_perm(bf.m, bf.row_leaf_ptr, bf.L, 2, 1)
    bf.col_perm = _subtree_perm(bf.n, bf.col_leaf_ptr, bf.L, 2, 2)
    return bf


def _fast_positions(blocks, per_peer, nrhs):
    """(element index in the region, tag) pairs of the half-slab exchange format: per peer
    [tile][half][block][16 rows][16 columns] (include/bfapply.h, bf_dist_slab_format 1)."""
    ntiles = (nrhs + 31) // 32
    out = []
    for qi in range(len(blocks) // per_peer):
        base = qi * ntiles * 2 * per_peer * 256
        for jt in range(ntiles):
            for half in range(2):
                for bi in range(per_peer):
                    b = int(blocks[qi * per_peer + bi])
                    for r in range(16):
                        for c16 in range(16):
                            col = jt * 32 + half * 16 + c16
                            pos = base + ((jt * 2 + half) * per_peer + bi) * 256 + r * 16 + c16
                            out.append((pos, b, r, col))
    return out


def _check_fast(h, op, nrhs, wb, so, ro, sc, rc, sblk, rblk, L, lc, p, rank, world):
    per = len(sblk) // world
    assert len(rblk) == len(sblk) == world * per
    assert all(c == ((nrhs + 31) // 32) * per * 512 for c in list(sc) + list(rc)), (sc, rc)
    tau, nu = sblk >> (L - lc), sblk & ((1 << (L - lc)) - 1)
    own = (nu >> (L - lc - p)) if op == "N" else (tau >> (lc - p))
    assert np.all(own == rank)
    dest = (tau >> (lc - p)) if op == "N" else (nu >> (L - lc - p))
    assert np.all(np.diff(dest) >= 0), "send region not grouped by destination"
    work = torch.zeros(wb, dtype=torch.uint8)
    send = work[so:so + sum(sc) * 16].view(torch.float64).view(-1, 2)
    for pos, b, r, col in _fast_positions(sblk, per, nrhs):
        send[pos, 0] = float(b)
        send[pos, 1] = 1000.0 * r + col
    h.exchange(work, op, nrhs)
    recv = work[ro:ro + sum(rc) * 16].view(torch.float64).view(-1, 2)
    for pos, b, r, col in _fast_positions(rblk, per, nrhs):
        assert recv[pos, 0] == float(b) and recv[pos, 1] == 1000.0 * r + col, (op, b, r, col)
    rt, rn = rblk >> (L - lc), rblk & ((1 << (L - lc)) - 1)
    mine = (rt >> (lc - p)) if op == "N" else (rn >> (L - lc - p))
    assert np.all(mine == rank), (op, "received blocks the rank does not own")


def _worker(rank, world, port, kind, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2007_00202_b200.dist import DistBFHandle
        bf = _case(kind)
        h = DistBFHandle(bf, rank, world, device=None)
        L, lc = bf.L, bf.lc
        p = world.bit_length() - 1
        nrhs = 3
        rank_row = bf.rank_row()[: 1 << L]          # r^lc_{tau,nu}, canonical order
        rank_col = bf.rank_col()[lc << L:]          # c^lc_{tau,nu}
        fmt = h.slab_format()
        assert fmt == (1 if kind == "fast" else 0), fmt
        for op in ("N", "C"):
            wb, so, ro, sc, rc = h.layout(op, nrhs)
            sblk, rblk = h.exchange_blocks(op)
            size = rank_row if op == "N" else rank_col
            if fmt == 1:  # the fused split exchanges at the pass-count-minimising level
                lx = h.exchange_level(op)
                assert p <= lx <= L - p
                _check_fast(h, op, nrhs, wb, so, ro, sc, rc, sblk, rblk, L, lx, p, rank, world)
                continue
            assert h.exchange_level(op) == lc
            tau, nu = sblk >> (L - lc), sblk & ((1 << (L - lc)) - 1)
            # sender owns the column subtree (op N) / row subtree (op C)
            own = (nu >> (L - lc - p)) if op == "N" else (tau >> (lc - p))
            assert np.all(own == rank), (op, "send blocks outside the rank's subtree")
            dest = (tau >> (lc - p)) if op == "N" else (nu >> (L - lc - p))
            assert np.all(np.diff(dest) >= 0), "send region not grouped by destination"
            for qq in range(world):
                assert sc[qq] == int(size[sblk[dest == qq]].sum()) * nrhs
            # tag every send element: re = block id, im = 1000 * row + col
            work = torch.zeros(wb, dtype=torch.uint8)
            send = work[so:so + sum(sc) * 16].view(torch.float64).view(-1, 2)
            k = 0
            for b in sblk:
                for r in range(int(size[b])):
                    for c in range(nrhs):
                        send[k, 0] = float(b)
                        send[k, 1] = 1000.0 * r + c
                        k += 1
            assert k == sum(sc)
            h.exchange(work, op, nrhs)
            recv = work[ro:ro + sum(rc) * 16].view(torch.float64).view(-1, 2)
            k = 0
            for b in rblk:
                for r in range(int(size[b])):
                    for c in range(nrhs):
                        assert recv[k, 0] == float(b) and recv[k, 1] == 1000.0 * r + c, (op, b, r, c)
                        k += 1
            assert k == sum(rc)
            rt, rn = rblk >> (L - lc), rblk & ((1 << (L - lc)) - 1)
            mine = (rt >> (lc - p)) if op == "N" else (rn >> (L - lc - p))
            assert np.all(mine == rank), (op, "received blocks the rank does not own")
            # every centre block is sent exactly once, over all ranks
            allb = [None] * world
            dist.all_gather_object(allb, sblk.tolist())
            flat = sorted(b for lst in allb for b in lst)
            assert flat == list(range(1 << L)), op
        # local rows: op N reads the column subtree, writes the row subtree
        ri, ro_, ui, uo = h.local_rows("N")
        w = 1 << (L - p)
        assert ri == bf.col_leaf_ptr[(rank + 1) * w] - bf.col_leaf_ptr[rank * w]
        assert ro_ == bf.row_leaf_ptr[(rank + 1) * w] - bf.row_leaf_ptr[rank * w]
        assert ui == bf.col_leaf_ptr[rank * w] and uo == bf.row_leaf_ptr[rank * w]
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # report, do not hang the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("kind", ["uniform", "ragged", "fast"])
@pytest.mark.parametrize("world", [2, 4])
def test_dist_exchange_gloo(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_dist_rejects_bad_layouts():
    from paper_2007_00202_b200.bfapply import BFError
    from paper_2007_00202_b200.dist import DistBFHandle
    bf = random_butterfly(L=4, leaf=2, r=2, seed=0)
    with pytest.raises(BFError) as e:
        DistBFHandle(bf, 0, 3, device=None)          # not a power of two
    assert e.value.code == -7
    with pytest.raises(BFError) as e:
        DistBFHandle(bf, 0, 8, device=None)          # p = 3 > min(lc, L - lc) = 2
    assert e.value.code == -7
    bf.col_perm = np.random.default_rng(0).permutation(bf.n)
    with pytest.raises(BFError) as e:
        DistBFHandle(bf, 0, 2, device=None)          # subtree not a contiguous user range
    assert e.value.code == -4
    h = DistBFHandle(random_butterfly(L=4, leaf=2, r=2, seed=0), 1, 2, device=None)
    with pytest.raises(BFError) as e:
        h.apply(torch.zeros((1, 16), dtype=torch.complex128))
    assert e.value.code == -8


def test_rhs_shard_partition():
    """The RHS-sharded HOD-BF layout (configs 3-4): every column owned by exactly one rank,
    contiguous, balanced to within one column."""
    from paper_2007_00202_b200.dist import rhs_shard
    for nrhs in (0, 1, 7, 64, 512, 513):
        for world in (1, 2, 3, 4, 8):
            parts = [rhs_shard(nrhs, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == nrhs
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
