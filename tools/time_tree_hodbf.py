"""Per-rank kernel time of the tree-partitioned HOD-BF (dist.TreeHODBF) on
config 3 or 4, measured on ONE GPU: for P = 2, 4, 8 every rank's launches (local HOD-BF,
column sides of the distributed levels, row sides + accumulate) run one after another with CUDA
events around each rank (no rank waits on another; the grouped send / receive is not timed,
its bytes per rank are reported).  max over ranks vs the single-GPU HOD-BF apply / P is the
compute side of the strong-scaling efficiency; the RHS-sharded layout (dist.ShardedHODBF) is
t1 / P per rank by construction.   python tools/time_tree_hodbf.py [cfg3|cfg4] [c128|c64]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bfinputs.configs import cfg3, cfg4  # noqa: E402
import paper_2007_00202_b200 as pkg  # noqa: E402
from paper_2007_00202_b200.dist import TreeHODBF  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    dts = sys.argv[2] if len(sys.argv) > 2 else "c128"
    dt = np.complex128 if dts == "c128" else np.complex64
    H, X = (cfg3 if name == "cfg3" else cfg4)(dt)
    nrhs = X.shape[1]
    h1 = pkg.HODBFHandle(H)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = h1.apply(Xd)
    t1 = timed(lambda: h1.apply(Xd, out=Y))
    del h1
    torch.cuda.empty_cache()
    res = {"config": name, "dtype": dts, "nrhs": nrhs, "single_gpu_ms": t1}
    Xt = X[H.perm]
    for P in (2, 4, 8):
        per, sent = [], []
        for g in range(P):
            t = TreeHODBF(H, g, P, 0)
            lo, hi = t.rows()
            Xl = torch.from_numpy(np.ascontiguousarray(Xt[lo:hi].T)).cuda()
            Yl = torch.empty_like(Xl)

            def run():
                t.local.apply(Xl, out=Yl)
                t.pre(Xl)
                t.post(Yl)
            per.append(timed(run))
            sent.append(sum(n for pl in t.exchange_plan("N", nrhs) for _, _, n in pl["sends"]))
            del t
            torch.cuda.empty_cache()
        res[f"P{P}"] = {"rank_ms": per, "max_ms": max(per), "eff_vs_single": t1 / P / max(per),
                        "send_bytes_per_rank": sent}
        print(json.dumps({f"P{P}": res[f"P{P}"]}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
