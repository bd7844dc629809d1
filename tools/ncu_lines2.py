"""Per-source-line share of executed instructions and stall samples of ONE launch of an ncu report, FP64 line
contractions folded into one row (dev helper): python tools/ncu_lines2.py rep.ncu-rep <launch index> [top]"""
import csv
import subprocess
import sys

rep, skip = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip",
                      str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
line, src, tot = None, {}, {}
for r in rows:
    if not r or len(r) < len(hdr) - 2:
        continue
    if r[0] not in ("", "Line No"):
        line = int(r[0])
        src[line] = r[1]
        continue
    try:
        v, w = float(r[ie].replace(",", "")), float(r[st].replace(",", ""))
    except ValueError:
        continue
    a = tot.setdefault(line, [0.0, 0.0])
    a[0] += v
    a[1] += w
T = sum(v[0] for v in tot.values())
S = sum(v[1] for v in tot.values())
print(f"warp instructions {T:.4g}, stall samples {S:.4g}")
eo = [v for ln, v in tot.items() if "lap_common" in src.get(ln, "") or ln < 100]
print(f"lines < 100 (lap_common.cuh eo_mv etc.): {sum(v[0] for v in eo) / T * 100:.1f}% instr {sum(v[1] for v in eo) / S * 100:.1f}% stalls")
for ln, v in sorted(tot.items(), key=lambda kv: -kv[1][1])[:top]:
    if ln < 100:
        continue
    print(f"{ln:5d} {v[0] / T * 100:5.1f}% {v[1] / S * 100:5.1f}%  {src[ln][:110]}")
