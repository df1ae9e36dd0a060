"""Summarise an ncu report: key throughput metrics, stall reasons, top SASS stall sites."""
import csv, re, subprocess, sys, collections

def raw(rep):
    """(header, rows) of the raw page; section prefixes ("SM_C.TriageCompute.") are stripped so
    every metric is found by its plain name."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = []
    for h in rows[0]:
        m = re.search(r"([a-z][a-z0-9]*__\S*)$", h)
        hdr.append(m.group(1) if m and m.group(1) not in hdr else h)
    return hdr, rows[2:]

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        # tensor pipe (sm_100 names): DMMA = mma.sync f64 (complex128), HMMA = mma.sync tf32 (complex64),
        # tc = tcgen05 (UTC*MMA)
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__cycles_active.avg",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]

def main(rep):
    hdr, rows = raw(rep)
    for r in rows:
        print("kernel:", r[hdr.index("Kernel Name")][:60])
        for k in KEYS:
            if k in hdr:
                print(f"  {k:75s} {r[hdr.index(k)]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("  stalls (cycles per issued instr):", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    data = [(int(x[si]) if x[si].isdigit() else 0, x[src].strip()) for x in rows[2:] if len(x) > si]
    tot = sum(d[0] for d in data) or 1
    op = collections.Counter()
    for s, t in data:
        op[t.split()[0] if t else "?"] += s
    print("  stall samples by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in op.most_common(10)))

if __name__ == "__main__":
    main(sys.argv[1])
