#!/usr/bin/env python
"""Benchmark: multi-RHS butterfly apply on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype c128|c64] [--op N|C]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference            # the CPU oracle arm (rank 0 only)

Workload (BASELINE.json configs[4], the config the metric's 1/2/4/8-GPU sweep is quoted
on): random-factor butterfly, n = m = 2^20, L = 14, lc = 7, leaf 64, rank 16, nrhs 32,
seed 1, complex128 (default) or complex64.  One step = one full apply Y = K X (all
SURVEY 8(a) rows a1-a5; a6 with --op C), inputs resident in HBM.  The factors (2.48 GB
c128 / 1.24 GB c64) are far larger than the 126 MB L2, so every step streams them from
HBM; no L2 flush is needed between steps.

value = algorithmic bytes / time (every factor entry an apply streams once + X read once + Y
written once; SURVEY 8(d) -- the centre B^{lc}, folded into R^{lc} at create, is not counted:
config.b_folded_entries), whole job.  Multi-GPU: the butterfly is split by column subtrees
(V, W, B) and row subtrees (R, U) with one NCCL all-to-all of the centre slabs; total
work is fixed (strong scaling).  Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "butterfly apply GB/s and RHS-columns/s, % of B200 HBM roofline, 1/2/4/8 GPUs"


def workload(args):
    return (f"cfg5: random-factor butterfly n=m=2^20, L=14, lc=7, leaf 64, r=16, nrhs={args.nrhs}, seed 1, "
            f"{args.dtype}, op {args.op}")


def _peaks():
    p = {"hbm_gbs": 6555.8, "source": "MEASURED_PEAKS.json"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p.update(json.load(f))
    except OSError:
        p = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "profiles", "pipe_peaks.json")) as f:
            p["pipes"] = json.load(f)
    except OSError:
        p["pipes"] = None
    return p


def ramp_clocks(ms: float = 150.0):
    """~150 ms of dummy device work (a streaming copy, none of the apply's kernels) before the
    warm-up steps, so that the SM clock is up from idle when they start: with small steps (nrhs 1:
    0.4 ms) W = 3 warm-up steps are ~1 ms, and the first timed steps then ran at idle clocks."""
    import time
    import torch
    a = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    t = time.perf_counter()
    while (time.perf_counter() - t) * 1e3 < ms:
        for _ in range(8):
            b.copy_(a)
        torch.cuda.synchronize()
    del a, b


class ClockSampler:
    """Polls NVML (SM clock + throttle reasons) on a thread during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device_index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0, "source": "nvml" if self.ok else "unavailable"}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


def cpu_threads():
    """Host cores this process may run on (os.sched_getaffinity; SURVEY 8(d) timing protocol)."""
    return len(os.sched_getaffinity(0))


def method_sample(bf, X, op, reps=1):
    """Time the level-by-level CPU apply (oracle/stagewise.py: the method on
    the host, all cores) on the WHOLE workload: one full apply per rep, measured, not
    extrapolated.  Returns (seconds per apply, threads)."""
    from oracle.stagewise import bf_apply_stagewise, host_threads
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        bf_apply_stagewise(bf, X, op)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), host_threads()


def cpu_model():
    """The host CPU's model name (SURVEY 8(d) timing protocol: cores and model with the oracle)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_sample(bf, X, nrows=(16, 128), centre=3):
    """Time the CPU oracle (sampled-row reconstruction) on rows of one
    centre node and extrapolate to the full apply with a two-point model
    T(rows) = setup + rows * per_row, full = 2^lc * setup + m * per_row."""
    import oracle
    w = bf.m >> bf.lc
    ts = []
    for r in nrows:
        rows = centre * w + np.arange(r)
        t0 = time.perf_counter()
        oracle.bf_rows_apply(bf, rows, X)
        ts.append(time.perf_counter() - t0)
    per_row = max((ts[1] - ts[0]) / (nrows[1] - nrows[0]), 1e-9)
    setup = max(ts[0] - nrows[0] * per_row, 0.0)
    full = (1 << bf.lc) * setup + bf.m * per_row
    return full, sum(ts), (f"oracle rows {nrows[0]} and {nrows[1]} of centre node {centre} "
                           f"({sum(ts):.1f} s total); full apply extrapolated as 2^lc*setup + m*per_row "
                           f"(setup {setup:.2f} s, per row {per_row*1e3:.2f} ms)")


def build_inputs(dtype_s, nrhs):
    from bfinputs.configs import cfg5
    dt = np.complex128 if dtype_s == "c128" else np.complex64
    return cfg5(dt, nrhs=nrhs)


# tensor-pipe work each dtype's kernels execute per complex multiply-add, and the measured peak
# of that pipe (profiles/pipe_peaks.json, tools/peaks.cu on this B200 pool)
PIPE = {"c128": ("dmma_sync_tflops", 6, "FP64 tensor pipe (mma.sync.m8n8k4.f64); 3M complex product = 3 real MACs "
                                        "= 6 flops per complex MAC"),
        "c64": ("tf32_mma_sync_tflops", 18, "TF32 tensor pipe (mma.sync.m16n8k8.tf32); 3M x 3xTF32 split = 9 real "
                                          "MACs = 18 flops per complex MAC")}
# The peak a contraction is measured against (task rule: its own dtype's peak = another dtype's
# measured peak x the guide's nominal ratio).  TF32: MEASURED_PEAKS bf16 x (1.1 / 2.25 PF, the
# guide's dense tf32 / bf16 nominals) -- the tcgen05-class TF32 rate of the chip, not the
# mma.sync rate the kernel can reach (kept beside it).  FP64: the guide states no FP64 figure,
# so the DMMA peak measured on this pool (tools/peaks.cu) stands.
TF32_OVER_BF16 = 1.1 / 2.25


def issued_cols(dtype, name, nrhs):
    """Right-hand-side columns the kernel's MMAs cover (the n-tile widths it instantiates): the
    window pass runs 8 columns per warp for nrhs <= 8 (complex128), one 16-column half for
    nrhs <= 16, else whole 32-column tiles; complex64's pass keeps 16 columns (its MMA's M) for
    nrhs <= 16.  The leaf kernels: 8 / 16 / 32-column variants likewise."""
    if dtype == "c128" and nrhs <= 8:
        return 8
    if nrhs <= 16:
        return 16 if (dtype == "c64" or nrhs > 8) else 8
    return 32 * ((nrhs + 31) // 32)


def dominant_roofline(dtype, name, rounds, mean, nrhs, cs, peaks):
    """Roofline of the kernel with the largest share of the step, from its per-launch CUDA-event
    times: algorithmic bytes (factor entries + user rows) against the HBM peak and the
    tensor-pipe work it executes against that pipe's measured peak; `bound` is the tighter one."""
    idx = [i for i, r in enumerate(rounds) if r["name"] == name]
    t = float(sum(mean[i] for i in idx)) * 1e-3 / len(idx)                 # s per launch
    b = sum((rounds[i]["factor_entries"] + (rounds[i]["user_rows_in"] + rounds[i]["user_rows_out"]) * nrhs) * cs
            for i in idx) / len(idx)                                        # bytes per launch
    key, fpc, note = PIPE[dtype]
    cols = issued_cols(dtype, name, nrhs)
    ent = sum(rounds[i]["factor_entries"] for i in idx) / len(idx)
    fl = ent * cols * fpc                                                     # pipe flops issued per launch
    method_fl = ent * nrhs * 8                                                # the method's own flops (8 per CMAC)
    sync_peak = ((peaks.get("pipes") or {}).get(key) or 0.0) * 1e12   # mma.sync rate measured on this pool
    if dtype == "c64" and peaks.get("bf16_tflops"):
        pipe_peak = peaks["bf16_tflops"] * TF32_OVER_BF16 * 1e12
        src = "MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 (B200_PROFILING.md tf32 / bf16 dense nominals)"
    else:
        pipe_peak = sync_peak
        src = "profiles/pipe_peaks.json (" + key + "; the guide states no FP64 figure)"
    hbm = {"achieved": b / t / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": b / t / 1e9 / peaks["hbm_gbs"],
           "peak_source": peaks.get("source")}
    ten = {"achieved": fl / t / 1e12, "peak": pipe_peak / 1e12, "unit": "TFLOP/s",
           "frac": (fl / t / pipe_peak) if pipe_peak else None, "peak_source": src, "work": note,
           "mma_sync_peak": sync_peak / 1e12,
           "frac_of_mma_sync_peak": (fl / t / sync_peak) if sync_peak else None}
    t_hbm = b / (peaks["hbm_gbs"] * 1e9)
    t_pipe = fl / pipe_peak if pipe_peak else 0.0
    main, other, bound = (ten, hbm, "tensor") if t_pipe > t_hbm else (hbm, ten, "hbm")
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dtype, {}).get(name)
    except (OSError, ValueError):
        pass
    return {"bound": bound, "achieved": main["achieved"], "peak": main["peak"], "unit": main["unit"],
            "frac": main["frac"], "traffic": traffic, "kernel": name, "launches_per_step": len(idx),
            "share_of_step": float(sum(mean[i] for i in idx) / mean.sum()), "peak_source": main["peak_source"],
            "alg_bytes_per_launch": b, "pipe_flops_per_launch": fl, "pipe_cols_issued": cols,
            "method_flops_per_launch": method_fl, "method_tflops": method_fl / t / 1e12,
            "other_bound": dict(other, bound="hbm" if bound == "tensor" else "tensor"),
            "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                            "(profiles/traffic.json)"}


def alg_entries(bf):
    """Factor entries an apply must stream: all of U, R, W, Vt.  The centre B^{lc} is folded into
    R^{lc} at create (R' = R B, the same shape as R), so its r x c entries per
    centre block are never read by an apply and are not counted (config 5: 4.19 M entries,
    1.9 % of the SURVEY 8(d) count, stated in config.b_folded_entries)."""
    return bf.nnz() - int(bf.B.data.size)


def alg_bytes(bf, nrhs, cs):
    return (alg_entries(bf) + (bf.m + bf.n) * nrhs) * cs


def make_config(args, bf, cs, world):
    """The config dict both arms print (same keys, same values)."""
    return {"workload": workload(args), "op": args.op, "nrhs": args.nrhs, "n": bf.n, "L": bf.L,
            "factor_entries": bf.nnz(), "alg_entries": alg_entries(bf), "b_folded_entries": int(bf.B.data.size),
            "alg_bytes_per_step": alg_bytes(bf, args.nrhs, cs),
            "l2": "inputs larger than L2 (factors %.2f GB >> 126 MB); no flush" % (bf.nnz() * cs / 1e9),
            "parallelism": "single GPU" if world == 1 else
            f"tree split over {world} GPUs (column subtrees -> "
            + {"p2p": "fused peer-memory exchange", "nccl": "NCCL all-to-all",
               "nccl-lib": "library-owned NCCL send / recv"}[args.exchange]
            + " -> row subtrees)"}


def run_reference(args):
    """The reference arm: the CPU oracle as it stands, on the host cores.  Each step is one FULL
    config-5 apply by the level-by-level oracle (oracle/stagewise.py; measured, nothing
    extrapolated).  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    bf, X = build_inputs(args.dtype, args.nrhs)
    cs = 16 if args.dtype == "c128" else 8
    ab = alg_bytes(bf, args.nrhs, cs)
    times = []
    threads = None
    for i in range(args.warmup + args.steps):
        t, threads = method_sample(bf, X, args.op)
        if i >= args.warmup:
            times.append(t)
    t = float(np.median(times))
    val = ab / t / 1e9
    sample = (f"one full config-5 apply (nrhs {args.nrhs}, op {args.op}) per step by oracle/stagewise.py "
              f"(level-by-level complex128 apply, {threads} threads); median of {args.steps} measured steps")
    line = {"metric": METRIC, "value": val, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": make_config(args, bf, cs, 1),
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cpu_threads(), "cpu_model": cpu_model(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--op", default="N", choices=["N", "C"])
    ap.add_argument("--nrhs", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p", "nccl-lib"],
                    help="N > 1: centre exchange by NCCL all-to-all (torch), fused into the kernel over peer "
                         "memory (torch symmetric memory; bf_dist_apply_pre_p2p), or by the library's own "
                         "NCCL communicator (bf_create_dist / bf_apply_dist: one C-ABI call per apply)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2007_00202_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = _peaks()
    bf, X = build_inputs(args.dtype, args.nrhs)
    cs = 16 if args.dtype == "c128" else 8
    ab = alg_bytes(bf, args.nrhs, cs)
    nrhs = args.nrhs
    stream = torch.cuda.current_stream()
    # BF_BENCH_SPLIT1=1: one GPU through the multi-GPU code path (DistBFHandle over a world of 1,
    # the exchange a local copy) -- a smoke of the N > 1 branch on a single device, not a bench line
    split = world > 1 or os.environ.get("BF_BENCH_SPLIT1") == "1"
    if not split:
        h = pkg.BFHandle(bf, local)
        rin, rout = (bf.n, bf.m) if args.op == "N" else (bf.m, bf.n)
        assert bf.m == bf.n, "config 5 is square: the same X block serves op N and op C"
        Xh = torch.from_numpy(np.ascontiguousarray(X.T))
        Xd = Xh.cuda()
        Yd = torch.empty((nrhs, rout), dtype=Xd.dtype, device="cuda")
        work = torch.empty(h.workspace_size(nrhs), dtype=torch.uint8, device="cuda")
        rounds = h.rounds(args.op)
        launches = len(rounds)

        def step(evs=None):
            if evs is None:
                h.apply(Xd, args.op, out=Yd, work=work)
            else:
                h.apply_events(Xd, evs, args.op, out=Yd, work=work)
    else:
        from paper_2007_00202_b200.dist import DistBFHandle, NcclComm
        h = DistBFHandle(bf, rank, world, local, comm=NcclComm(local) if args.exchange == "nccl-lib" else None)
        if args.exchange == "p2p":
            h.enable_p2p(args.nrhs, args.op)
        Xloc = h.local_input(X, args.op)
        Xd = torch.from_numpy(np.ascontiguousarray(Xloc.T)).cuda()
        Yd = h.empty_output(nrhs, args.op)
        launches = h.launches(args.op)
        rounds = None

        def step(evs=None):
            h.apply(Xd, args.op, out=Yd)
    ramp_clocks()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # the timed region: K plain applies, exactly as a user calls them (no events between the
    # launches: an event record between two kernels would serialise the programmatic dependent
    # launch overlap of the fused path)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for k in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps
    # per-launch durations (N = 1), live in this run: the same K steps again with an event
    # between every two launches (one set per step)
    ev_sets = None
    ms_evented = None
    if rounds is not None:
        ev_sets = [[torch.cuda.Event(enable_timing=True) for _ in range(len(rounds) + 1)] for _ in range(args.steps)]
        for s in ev_sets:
            for e in s:
                e.record(stream)
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            step(ev_sets[k])
        t1.record(stream)
        torch.cuda.synchronize()
        ms_evented = t0.elapsed_time(t1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = ab / (ms * 1e-3) / 1e9

    roofline = None
    per_round = None
    if ev_sets is not None:
        times = np.array([[s[i].elapsed_time(s[i + 1]) for i in range(len(rounds))] for s in ev_sets])
        mean = times.mean(axis=0)
        per_round = []
        by_kernel = {}
        for i, r in enumerate(rounds):
            b = (r["factor_entries"] + (r["user_rows_in"] + r["user_rows_out"]) * nrhs) * cs
            per_round.append({"round": i, "kernel": r["name"], "ms": float(mean[i]), "alg_bytes": int(b),
                              "gbs": b / (mean[i] * 1e-3) / 1e9})
            k = by_kernel.setdefault(r["name"], [0.0, 0, 0])
            k[0] += mean[i]
            k[1] += b
            k[2] += 1
        name, (kms, kb, kn) = max(by_kernel.items(), key=lambda kv: kv[1][0])
        roofline = dominant_roofline(args.dtype, name, rounds, mean, nrhs, cs, peaks)
        roofline["kernels"] = {k: {"ms_per_step": v[0], "launches_per_step": v[2], "alg_bytes_per_step": v[1]}
                               for k, v in by_kernel.items()}
    elif split:
        # N > 1: per rank, the whole split apply (its leaf / pass launches and the exchange) against
        # the HBM roofline of one GPU -- each rank streams 1/N of the factors and its subtrees' rows
        # (per-launch events are not exposed by the split's pre / post calls, so this is step-level)
        per_rank = ab / world
        ach = per_rank / (ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / peaks["hbm_gbs"], "traffic": None, "kernel": "split apply per rank (step-level)",
                    "alg_bytes_per_rank": per_rank, "peak_source": peaks.get("source"),
                    "note": "max over ranks of the step time; algorithmic bytes / N per rank"}

    e2e = None
    if not args.no_e2e and not split:
        Xp = Xh.pin_memory()
        Yp = torch.empty((nrhs, Yd.shape[1]), dtype=Xd.dtype).pin_memory()
        wh = torch.empty(max(h.workspace_size_host(nrhs, args.op), 1), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            h.apply_host(Xp, args.op, out=Yp, work=wh)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(3, min(args.steps, 10))
        e0.record(stream)
        for _ in range(ke):
            h.apply_host(Xp, args.op, out=Yp, work=wh)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / ke
        e2e = {"value": ab / (ems * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(Xp.numel() * cs), "d2h_bytes_per_step": int(Yp.numel() * cs),
               "api": "bf_apply_host (pinned host X/Y; every step's H2D and D2H inside the timed region, "
                      "consecutive calls overlap one's D2H with the next one's H2D on the handle's copy streams)"}
    elif not args.no_e2e and split:
        e2e = h.time_e2e(X_loc_host=Xd.cpu(), op=args.op, steps=max(3, min(args.steps, 10)), alg_bytes=ab)

    cpu = cpu_m = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        full, spent, sample = oracle_sample(bf, X)
        cpu = {"value": ab / full / 1e9, "unit": "GB/s", "cores": cpu_threads(), "cpu_model": cpu_model(),
               "kind": "oracle", "extrapolated": True,
               "sample": "dense-definition oracle (oracle/dense.py, Eq. 3.1-3.2 per sampled row): " + sample}
        tm, thr = method_sample(bf, X, args.op)
        cpu_m = {"value": ab / tm / 1e9, "unit": "GB/s", "cores": thr, "cpu_model": cpu_model(), "kind": "method",
                 "extrapolated": False, "ms_per_step": tm * 1e3,
                 "sample": f"one full config-5 apply (nrhs {nrhs}, op {args.op}) by the level-by-level CPU apply "
                           f"(oracle/stagewise.py, SURVEY C2 step 6), {thr} threads, measured"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
                "config": make_config(args, bf, cs, world),
                "rhs_cols_per_s": nrhs / (ms * 1e-3), "hbm_frac": value / peaks["hbm_gbs"],
                "roofline": roofline, "cpu_baseline": cpu, "cpu_baseline_method": cpu_m, "e2e": e2e,
                "gpu_launches": launches * args.steps, "clocks": clk.summary(), "per_round": per_round,
                "ms_per_step_evented": ms_evented}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
