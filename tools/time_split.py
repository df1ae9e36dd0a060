"""Per-rank kernel time of the multi-GPU split of config 5, measured on ONE GPU: for P = 1, 2,
4, 8 every rank's pre (leaf-in + W passes) and post (R passes + leaf-out) launches run one
after another (CUDA events around each rank's launches; no rank waits on another; the
all-to-all is not timed here).  max over ranks of (pre + post) vs the single-GPU apply / P
is the compute side of the strong-scaling efficiency.   python tools/time_split.py [c128|c64]"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bfinputs.configs import cfg5  # noqa: E402
from paper_2007_00202_b200.bfapply import OPS, lib  # noqa: E402
from paper_2007_00202_b200.dist import DistBFHandle  # noqa: E402
import paper_2007_00202_b200 as pkg  # noqa: E402


def main():
    dts = sys.argv[1] if len(sys.argv) > 1 else "c128"
    dt = np.complex128 if dts == "c128" else np.complex64
    bf, X = cfg5(dt)
    nrhs = X.shape[1]
    h1 = pkg.BFHandle(bf)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = h1.apply(Xd)
    for _ in range(3):
        h1.apply(Xd, out=Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        h1.apply(Xd, out=Y)
    e1.record()
    torch.cuda.synchronize()
    t1 = e0.elapsed_time(e1) / 10
    del h1
    res = {"dtype": dts, "single_gpu_ms": t1}
    for P in (1, 2, 4, 8):
        per = []
        for g in range(P):
            h = DistBFHandle(bf, g, P, 0)
            assert h.slab_format() == 1
            ri, ro, ui, uo = h.local_rows("N")
            Xl = torch.from_numpy(np.ascontiguousarray(X[ui:ui + ri].T)).cuda()
            Yl = torch.empty((nrhs, ro), dtype=Xl.dtype, device="cuda")
            w = torch.zeros(h.layout("N", nrhs)[0], dtype=torch.uint8, device="cuda")

            def run():
                assert lib().bf_dist_apply_pre(h.h, OPS["N"], nrhs, C.c_void_p(Xl.data_ptr()), ri,
                                               C.c_void_p(w.data_ptr()), w.numel(), None) == 0
                assert lib().bf_dist_apply_post(h.h, OPS["N"], nrhs, C.c_void_p(Yl.data_ptr()), ro,
                                                C.c_void_p(w.data_ptr()), w.numel(), None) == 0
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                run()
            e1.record()
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1) / 10)
            del h, w
            torch.cuda.empty_cache()
        res[f"P{P}"] = {"rank_ms": per, "max_ms": max(per), "eff_vs_single": t1 / P / max(per)}
        print(json.dumps({f"P{P}": res[f"P{P}"]}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
