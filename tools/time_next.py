"""Time the SURVEY 8(f) "next" rows on one B200 and print one JSON object per line:
  NEXT-2 bf_random_matvec: recompression of (a) a config-5-shaped random butterfly at L = 10 through
         its own apply and (b) the config-2 Helmholtz operator's normal product A^H A;
  NEXT-3 hodbf_invert: a Helmholtz HOD-BF of a 64 x 64 plane (config-3 recipe at 1/4 size);
  NEXT-4 bf_mf_solve: the solve-phase sweep over a depth-3 synthetic assembly tree, nrhs 1 / 8 / 32.
python tools/time_next.py [next2 next3 next4]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_00202_b200 as pkg  # noqa: E402
from paper_2007_00202_b200 import construct as cx  # noqa: E402
from bfinputs import random_butterfly, random_rhs  # noqa: E402


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X).T)).cuda()


def probe_err(apply_a, apply_b, n, k=8, seed=0):
    X = dev(random_rhs(n, k, seed=seed))
    Ya, Yb = apply_a(X), apply_b(X)
    torch.cuda.synchronize()
    return float(torch.linalg.norm(Ya - Yb) / torch.linalg.norm(Yb))


def next2():
    bf = random_butterfly(L=10, leaf=64, r=16, seed=1)
    h = pkg.BFHandle(bf)
    op = cx.Operator(bf.m, bf.n, np.complex128, [(1.0, [(h, "N")], 0, 0)])
    t0 = time.perf_counter()
    res = cx.random_matvec(op, bf.m, bf.n, bf.L, bf.row_leaf_ptr, bf.col_leaf_ptr, eps=1e-12, rank_max=20,
                           oversample=8, seed=3)
    wall = time.perf_counter() - t0
    err = probe_err(lambda X: res.handle.apply(X), lambda X: h.apply(X), bf.n)
    print(json.dumps({"row": "NEXT-2", "case": "cfg5-shaped random butterfly L=10 (n=65536, r=16) via its apply",
                      "wall_s": wall, "stats": res.stats, "probe_rel_err": err}), flush=True)
    from bfinputs.configs import cfg2
    A, _ = cfg2()
    hA = pkg.BFHandle(A)
    op = cx.Operator(A.n, A.n, np.complex128, [(1.0, [(hA, "N"), (hA, "C")], 0, 0)])
    t0 = time.perf_counter()
    res = cx.random_matvec(op, A.n, A.n, A.L, A.col_leaf_ptr, A.col_leaf_ptr, A.col_perm, A.col_perm, eps=1e-6,
                           rank_max=256, oversample=16, seed=5)
    wall = time.perf_counter() - t0
    err = probe_err(lambda X: res.handle.apply(X), lambda X: op.apply(X), A.n)
    print(json.dumps({"row": "NEXT-2", "case": "config-2 Helmholtz A^H A (n=4096, L=6), eps 1e-6",
                      "wall_s": wall, "stats": res.stats, "probe_rel_err": err}), flush=True)


def next3():
    from bfinputs.configs import helmholtz_plane_hodbf
    H = helmholtz_plane_hodbf(64, 64, 10.0, 1e-4)
    hh = pkg.HODBFHandle(H)
    for dense_max in (256, 0):
        t0 = time.perf_counter()
        inv = cx.HODBFInverse(H, eps=1e-8, rank_max=96, dense_max=dense_max)
        wall = time.perf_counter() - t0
        X = dev(random_rhs(H.n, 8, seed=1))
        R = hh.apply(inv.apply(X))
        torch.cuda.synchronize()
        res = float(torch.linalg.norm(R - X) / torch.linalg.norm(X))
        # apply time at nrhs 1 / 32
        times = {}
        for k in (1, 32):
            Xk = dev(random_rhs(H.n, k, seed=2))
            Y = inv.apply(Xk)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                inv.apply(Xk, out=Y)
            e1.record()
            torch.cuda.synchronize()
            times[k] = e0.elapsed_time(e1) / 10
        print(json.dumps({"row": "NEXT-3", "case": f"Helmholtz HOD-BF 64x64 plane (n={H.n}, LH={H.LH}), eps 1e-8, "
                          f"dense_max {dense_max}", "wall_s": wall, "stats": inv.stats,
                          "residual": res, "inverse_entries": inv.factor_entries, "node_butterflies": inv.nbutterflies,
                          "apply_ms": times}), flush=True)


def next4():
    from bfinputs.fronts import synthetic_fronts
    fronts, N = synthetic_fronts(depth=3, nx_leaf=16, seed=1)
    t0 = time.perf_counter()
    mf = cx.MFSolver(fronts, N, eps=1e-8, rank_max=96, dense_max=256)
    build = time.perf_counter() - t0
    out = {"row": "NEXT-4", "case": f"depth-3 assembly tree, {len(fronts)} fronts, N={N}", "build_s": build}
    for k in (1, 8, 32):
        B = dev(random_rhs(N, k, seed=k))
        X = mf.solve(B)
        work = torch.empty(mf.workspace_size(k), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            mf.solve(B, out=X, work=work)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            mf.solve(B, out=X, work=work)
        e1.record()
        torch.cuda.synchronize()
        out[f"solve_ms_nrhs{k}"] = e0.elapsed_time(e1) / 20
        # the sweep is asynchronous with a caller workspace: capture it once into a CUDA graph and
        # replay (removes the per-launch host cost of the ~hundreds of small launches)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            mf.solve(B, out=X, work=work)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                mf.solve(B, out=X, work=work)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[f"solve_graph_ms_nrhs{k}"] = e0.elapsed_time(e1) / 20
        Xg = X.clone()
        mf.solve(B, out=X, work=work)
        torch.cuda.synchronize()
        out[f"graph_equals_direct_nrhs{k}"] = bool(torch.equal(Xg, X))
    out["factor_entries"] = int(sum(inv.factor_entries for inv in mf.inv) +
                                sum(b.info["factor_entries"] for b in mf.bfs))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["next2", "next3", "next4"]
    for w in which:
        globals()[w]()
