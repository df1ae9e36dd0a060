import time, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
t = time.time()
from bfinputs.configs import cfg5
import paper_2007_00202_b200 as pkg
dt = np.complex128 if sys.argv[1] == "c128" else np.complex64
bf, X = cfg5(dt)
print("gen", time.time() - t, flush=True)
t = time.time()
h = pkg.BFHandle(bf)
print("create", time.time() - t, h.info, flush=True)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
torch.cuda.synchronize()
for i in range(3):
    t = time.time()
    Y = h.apply(Xd)
    torch.cuda.synchronize()
    print("apply", i, time.time() - t, flush=True)
