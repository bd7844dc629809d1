"""Per (file, line) share of executed instructions and stall samples of one launch of an ncu report, sorted by
stall samples (dev helper): python tools/ncu_lines3.py rep.ncu-rep [launch index] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip",
                      str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cur, fil, tot, src = None, None, {}, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fil = r[1].split("/")[-1]
        continue
    if r[0] not in ("", "Line No"):
        if r[0].isdigit():
            cur = (fil, int(r[0]))
            src[cur] = r[1]
        continue
    if len(r) > ie and cur is not None:
        try:
            v, w = float(r[ie].replace(",", "")), float(r[st].replace(",", ""))
        except ValueError:
            continue
        a = tot.setdefault(cur, [0.0, 0.0])
        a[0] += v
        a[1] += w
T = sum(v[0] for v in tot.values())
S = sum(v[1] for v in tot.values())
print(f"warp instructions {T:.4g}, stall samples {S:.4g}")
byfile = {}
for (f, _), v in tot.items():
    b = byfile.setdefault(f, [0.0, 0.0])
    b[0] += v[0]
    b[1] += v[1]
print("per file (instr %, stall %):", {k: (round(v[0] / T * 100, 1), round(v[1] / S * 100, 1)) for k, v in byfile.items()})
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0][:14]:14s} {k[1]:5d} {v[0] / T * 100:5.1f}% {v[1] / S * 100:5.1f}%  {src[k][:100]}")
