"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per launch) into per-launch lines and
each kernel's share of the step.  usage: python tools/ncu_launches.py launches.csv "title" > summary.txt"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
i_id, i_name, i_metric, i_val = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
i_unit = hdr.index("Metric Unit")
launch = {}
for r in rows[1:]:
    d = launch.setdefault(int(r[i_id]), {"name": r[i_name]})
    v = float(r[i_val].replace(",", ""))
    u = r[i_unit]
    if r[i_metric] == "gpu__time_duration.sum":
        d["us"] = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    else:
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        d["rd" if "read" in r[i_metric] else "wr"] = v * scale
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print("# ncu --clock-control none, serialised cold-cache replay: compare SHARES of the step, not absolute times")
print("id kernel time_us dram_read_MB dram_write_MB")
tot = sum(d.get("us", 0) for d in launch.values())
agg = {}
for k in sorted(launch):
    d = launch[k]
    nm = d["name"].split("(")[0].replace("void ", "").replace("cnrx::<unnamed>::", "").replace("<unnamed>::", "")
    print(f"{k} {nm[:48]:48s} {d.get('us', 0):9.1f} {d.get('rd', 0):9.1f} {d.get('wr', 0):9.1f}")
    a = agg.setdefault(nm, [0.0, 0.0, 0])
    a[0] += d.get("us", 0)
    a[1] += d.get("rd", 0) + d.get("wr", 0)
    a[2] += 1
print(f"# total {tot:.1f} us")
for nm, (us, mb, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"#   {nm[:48]:48s} x{n}  {us:9.1f} us  {100 * us / tot:5.1f} %  {mb / max(us, 1e-9):6.2f} TB/s")
