"""Write profiles/traffic.json: average DRAM bytes (read + write) per launch of every fast-path
kernel, from ncu CSV logs (`--metrics dram__bytes_read.sum,dram__bytes_write.sum --csv`).

    python tools/make_traffic.py c128=gpurun_out/traffic_c128.csv c64=gpurun_out/traffic_c64.csv
"""
import collections
import csv
import json
import os
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name, dtype):
    if "k_bf_pass" in name:
        return f"k_bf_pass<{dtype}>"
    if "k_leaf" in name:
        return f"k_leaf<{dtype},{'in' if re.search(r'\(int\)0>|, 0>', name) else 'out'}>"
    return name


def parse(path, dtype):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    iK, iM, iU, iV, iI = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(float)
    names = {}
    for r in rows[1:]:
        if r[iM] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[r[iI]] += float(r[iV].replace(",", "")) * UNIT.get(r[iU], 1)
            names[r[iI]] = short(r[iK], dtype)
    agg = collections.defaultdict(list)
    for i, v in per.items():
        agg[names[i]].append(v)
    return {k: sum(v) / len(v) for k, v in agg.items()}


def main():
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    res = {}
    for a in sys.argv[1:]:
        dt, path = a.split("=", 1)
        res[dt] = parse(path, dt)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
