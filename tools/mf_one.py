"""One multifrontal sweep (depth-3 synthetic tree, nrhs 1) after warm-up: for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00202_b200 import construct as cx  # noqa: E402
from bfinputs import random_rhs  # noqa: E402
from bfinputs.fronts import synthetic_fronts  # noqa: E402

fronts, N = synthetic_fronts(depth=3, nx_leaf=16, seed=1)
mf = cx.MFSolver(fronts, N, eps=1e-8, rank_max=96, dense_max=256)
B = torch.from_numpy(np.ascontiguousarray(random_rhs(N, 1, seed=1).T)).cuda()
X = mf.solve(B)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
mf.solve(B, out=X)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
