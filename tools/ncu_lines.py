"""Per-CUDA-source-line totals from an ncu report's mixed source page (dev helper).

python tools/ncu_lines.py rep.ncu-rep [column ...]  -> lines sorted by the first column
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
cols = sys.argv[2:] or ["L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "Warp Stall Sampling (All Samples)"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
idx = [hdr.index(c) for c in cols]
src = {}
tot = {}
line = None
for r in rows:
    if not r or len(r) < len(hdr) - 2:
        continue
    if r[0] not in ("", "Line No"):
        line = int(r[0])
        src[line] = r[1]
        continue
    if r[0] == "" and line is not None:
        t = tot.setdefault(line, [0.0] * len(cols))
        for j, i in enumerate(idx):
            try:
                t[j] += float(r[i].replace(",", ""))
            except ValueError:
                pass
grand = [sum(t[j] for t in tot.values()) for j in range(len(cols))]
print(" | ".join(f"{c}: {g:.4g}" for c, g in zip(cols, grand)))
for ln, t in sorted(tot.items(), key=lambda kv: -kv[1][0])[:40]:
    if t[0] <= 0:
        break
    print(f"{ln:5d} " + " ".join(f"{v / max(g, 1) * 100:6.1f}%" for v, g in zip(t, grand)) + "  " + src[ln][:90])
