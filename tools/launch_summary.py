"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel (dev helper).

python tools/launch_summary.py launches.csv [header lines ...]
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ii], {"name": r[ki].split("(")[0]})
    d[r[mi]] = float(r[vi].replace(",", ""))
for line in sys.argv[2:]:
    print(line)
per = OrderedDict()
for d in launch.values():
    p = per.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
    p[0] += 1
    p[1] += d.get("gpu__time_duration.sum", 0.0) / 1e6
    p[2] += d.get("dram__bytes_read.sum", 0.0) / 1e9
    p[3] += d.get("dram__bytes_write.sum", 0.0) / 1e9
tot = sum(p[1] for p in per.values())
print(f"\n{'kernel':72s} {'launches':>8s} {'ms total':>9s} {'ms/launch':>10s} {'share':>6s} {'GB rd/l':>8s} {'GB wr/l':>8s}")
for k, p in per.items():
    print(f"{k[:72]:72s} {p[0]:8d} {p[1]:9.3f} {p[1] / p[0]:10.4f} {p[1] / tot * 100:5.1f}% {p[2] / p[0]:8.3f} {p[3] / p[0]:8.3f}")
print("\nlaunch sequence:")
for d in launch.values():
    print(f"  {d['name'][:70]:70s} {d.get('gpu__time_duration.sum', 0) / 1e6:8.4f} ms  rd {d.get('dram__bytes_read.sum', 0) / 1e9:6.3f} GB"
          f"  wr {d.get('dram__bytes_write.sum', 0) / 1e9:6.3f} GB")
