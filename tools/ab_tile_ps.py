"""A/B of the complex128 transposed tile kernel's presummed chunks (BF_TILE_PS) on configs 2-4,
in one process (the knob is read per launch): python tools/ab_tile_ps.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_00202_b200 as pkg  # noqa: E402
from bfinputs.configs import cfg2, cfg3, cfg4  # noqa: E402
from tools.time_configs import timeit  # noqa: E402

cases = []
bf, X = cfg2(np.complex128)
cases.append(("cfg2", pkg.BFHandle(bf), X))
H, X = cfg3(np.complex128)
cases.append(("cfg3", pkg.HODBFHandle(H), X))
H, X = cfg4(np.complex128, proxy_cap=512)
cases.append(("cfg4", pkg.HODBFHandle(H), X))
for rep in range(2):
    for v in ("1", "0"):
        os.environ["BF_TILE_PS"] = v
        for name, h, X in cases:
            r = {op: timeit(h, X, op, X.shape[1], 1.0) for op in "NC"}
            print(f"rep {rep} PS={v} {name} N {r['N']['ms']:.4f} C {r['C']['ms']:.4f} "
                  f"rounds N {[d['ms'] for d in r['N']['detail']]}", flush=True)
