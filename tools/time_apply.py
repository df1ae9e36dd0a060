"""Plain apply loop on config 5 (no per-launch events between kernels): ms per apply, best of
5 runs of 20 applies.   python tools/time_apply.py [c128|c64] [N|C] [nrhs]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bfinputs.configs import cfg5  # noqa: E402
import paper_2007_00202_b200 as pkg  # noqa: E402


def main():
    dts = sys.argv[1] if len(sys.argv) > 1 else "c128"
    op = sys.argv[2] if len(sys.argv) > 2 else "N"
    nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    bf, X = cfg5(np.complex128 if dts == "c128" else np.complex64, nrhs=nrhs)
    h = pkg.BFHandle(bf)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = h.apply(Xd, op)
    work = torch.empty(h.workspace_size(X.shape[1]), dtype=torch.uint8, device="cuda")
    for _ in range(5):
        h.apply(Xd, op, out=Y, work=work)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for _ in range(20):
            h.apply(Xd, op, out=Y, work=work)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
    print(f"{dts} op {op} nrhs {nrhs}: {best:.4f} ms/apply")


if __name__ == "__main__":
    main()
