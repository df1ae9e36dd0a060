"""bf_extract (extract_BF as a partial matvec) on the config-5 butterfly and
hodbf_extract on the config-3 HOD-BF: wall time per call (synchronous: host planning of
the touched blocks + uploads + kernels) for typical sub-block shapes, next to the full apply.
    python tools/time_extract.py [c128|c64]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bfinputs.configs import cfg5  # noqa: E402
import paper_2007_00202_b200 as pkg  # noqa: E402


def main():
    dts = sys.argv[1] if len(sys.argv) > 1 else "c128"
    bf, X = cfg5(np.complex128 if dts == "c128" else np.complex64)
    h = pkg.BFHandle(bf)
    rng = np.random.default_rng(0)
    leaf = int(bf.row_leaf_ptr[1] - bf.row_leaf_ptr[0])
    cases = {
        "one leaf block 64x64": (np.arange(5 * leaf, 6 * leaf), np.arange(900 * leaf, 901 * leaf)),
        "16 x 16 scattered": (rng.integers(0, bf.m, 16), rng.integers(0, bf.n, 16)),
        "256 x 256 scattered": (rng.integers(0, bf.m, 256), rng.integers(0, bf.n, 256)),
        "4 leaves x 4 leaves (256 x 256)": (np.arange(64 * leaf, 68 * leaf), np.arange(3000 * leaf, 3004 * leaf)),
    }
    res = {"dtype": dts}
    for name, (I, J) in cases.items():
        h.extract(I, J)  # first call also builds the cached inverse perms
        t = []
        for _ in range(5):
            t0 = time.perf_counter()
            h.extract(I, J)
            t.append(time.perf_counter() - t0)
        res[name] = {"ms": 1e3 * float(np.median(t)), "entries": len(I) * len(J)}
        print(name, json.dumps(res[name]), flush=True)
    # extract_HODBF on config 3 (c128): a leaf block, a 256 x 256 block of 4 x 4 leaves, scattered
    from bfinputs.configs import cfg3
    H, _ = cfg3(np.complex128)
    hh = pkg.HODBFHandle(H)
    lp = H.leaf_ptr
    hcases = {
        "cfg3 HOD-BF one leaf block 64x64": (H.perm[lp[7]:lp[8]], H.perm[lp[7]:lp[8]]),
        "cfg3 HOD-BF 4 x 4 leaves off-diagonal (256 x 256)": (H.perm[lp[0]:lp[4]], H.perm[lp[200]:lp[204]]),
        "cfg3 HOD-BF 256 x 256 scattered": (rng.integers(0, H.n, 256), rng.integers(0, H.n, 256)),
    }
    for name, (I, J) in hcases.items():
        hh.extract(I, J)
        t = []
        for _ in range(5):
            t0 = time.perf_counter()
            hh.extract(I, J)
            t.append(time.perf_counter() - t0)
        res[name] = {"ms": 1e3 * float(np.median(t)), "entries": len(I) * len(J)}
        print(name, json.dumps(res[name]), flush=True)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = h.apply(Xd)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        h.apply(Xd, out=Y)
    torch.cuda.synchronize()
    res["full apply nrhs 32 (ms)"] = 1e3 * (time.perf_counter() - t0) / 10
    print(json.dumps(res))


if __name__ == "__main__":
    main()
