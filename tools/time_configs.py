"""Time the apply on BASELINE.json configs 1-3 (generic batched path: ragged ranks, HOD-BF) and
print per-round kernel times.  python tools/time_configs.py [cfg ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_00202_b200 as pkg  # noqa: E402
from bfinputs.configs import cfg1, cfg2, cfg3, cfg4  # noqa: E402


def timeit(h, X, op, nrhs, alg, steps=20):
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = h.apply(Xd, op)
    rounds = h.rounds(op)
    for _ in range(3):
        h.apply(Xd, op, out=Y)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(rounds) + 1)] for _ in range(steps)]
    for s in evs:  # torch creates the CUDA event on first record
        for e in s:
            e.record()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for k in range(steps):
        h.apply(Xd, op, out=Y)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    for k in range(steps):
        h.apply_events(Xd, evs[k], op, out=Y)
    torch.cuda.synchronize()
    per = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(len(rounds))] for e in evs]).mean(0)
    detail = [{"ms": round(float(per[i]), 4), "tasks": r["ntasks"], "entries": r["factor_entries"],
               "tflops": round(8 * r["factor_entries"] * nrhs / (per[i] * 1e-3) / 1e12, 2)} for i, r in enumerate(rounds)]
    gr = h.graph(Xd.clone(), op)  # the same apply replayed from a CUDA graph (launch-bound configs)
    gr.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms_graph = e0.elapsed_time(e1) / steps
    return {"ms": ms, "ms_graph": ms_graph, "GB/s": alg / ms / 1e6, "rounds": len(rounds), "detail": detail,
            "by_kernel": {n: round(float(sum(per[i] for i, r in enumerate(rounds) if r["name"] == n)), 4)
                          for n in sorted({r["name"] for r in rounds})}}


def main():
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
    out = {}
    for c in which:
        for dt in ([np.complex128, np.complex64] if c == "cfg3" else [np.complex128]):
            cs = 16 if dt == np.complex128 else 8
            if c in ("cfg3", "cfg4"):
                H, X = cfg3(dt) if c == "cfg3" else cfg4(dt, proxy_cap=512)
                h = pkg.HODBFHandle(H)
                nnz = H.nnz()
                n = m = H.n
            else:
                bf, X = (cfg1 if c == "cfg1" else cfg2)(dt)
                h = pkg.BFHandle(bf)
                nnz, n, m = bf.nnz(), bf.n, bf.m
            nrhs = X.shape[1]
            alg = (nnz + (n + m) * nrhs) * cs
            key = f"{c}-{'c128' if cs == 16 else 'c64'}"
            out[key] = {op: timeit(h, X, op, nrhs, alg) for op in "NC"}
            out[key]["factor_entries"] = int(nnz)
            out[key]["nrhs"] = int(nrhs)
            print(key, json.dumps(out[key]), flush=True)
    return out


if __name__ == "__main__":
    main()
