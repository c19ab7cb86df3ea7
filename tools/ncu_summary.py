"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv) per kernel: launches, mean duration, share of the listed time, mean DRAM bytes per launch.
Writes the per-kernel DRAM traffic that bench.py reports as roofline.traffic (profiles/ncu_traffic.json).

usage: python tools/ncu_summary.py gpurun_out/ncu_launches.csv [out_prefix]"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# library launch names (cnrx_launch_name) <- demangled ncu kernel names
ALIASES = [(r"conv_ws64_kernel", "conv_ws64_kernel"), (r"conv_tc_kernel<(\d+), ?(\d+), ?(\d+)>", r"conv_tc_kernel<\1,\2,\3>"),
           (r"head_tma_kernel", "head_tma_kernel"), (r"featurize_kernel<1", "featurize_kernel<plane>"),
           (r"pw_fold_kernel", "pw_fold_kernel<head>")]


def short(name):
    for pat, rep in ALIASES:
        m = re.search(pat, name)
        if m:
            return m.expand(rep)
    return name.split("(")[0][:60]


def main():
    path = sys.argv[1]
    prefix = sys.argv[2] if len(sys.argv) > 2 else None
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if r[0] == "ID")
    H = rows[hdr]
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        d = dict(zip(H, r))
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        names[d["ID"]] = short(d["Kernel Name"])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':32s} {'launches':>8s} {'mean us':>9s} {'share':>7s} {'DRAM MB/launch':>15s} {'GB/s':>8s}"]
    traffic = {}
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:32s} {n:8d} {t / n / 1e3:9.1f} {t / total:7.1%} {b / n / 1e6:15.1f} {b / t:8.0f}")
        traffic[k] = b / n
    print("\n".join(lines))
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump({"source": os.path.basename(path), "unit": "bytes per launch (dram read + write)", **traffic}, f,
                  indent=1)
    if prefix:
        with open(prefix + "_summary.txt", "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
