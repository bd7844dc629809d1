#!/bin/bash
# Median kernel durations per kernel name over a few ops under ncu (cold-cache, serialised: stable to ~0.2 %,
# unlike event timing on a shared box).  Usage: tools/ncu_times.sh [kernel regex] [command ...]   (dev helper)
RE=${1:-lap_plane_kernel|slot_fixup}
shift
CMD=${@:-python tools/time_yt.py c5 2}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$RE" -c 60 --csv $CMD 2>/dev/null | python -c "
import csv, sys, statistics
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
h = rows[0]; k, v, u = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
d = {}
for r in rows[1:]:
    t = float(r[v].replace(',', '')) * {'ns': 1e-6, 'us': 1e-3, 'ms': 1.0, 'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0}.get(r[u], 1.0)
    d.setdefault(r[k].split('(')[0], []).append(t)
for n, ts in d.items():
    print(f'{n[-62:]:62s} n={len(ts):3d} median {statistics.median(ts):.4f} ms  min {min(ts):.4f}')
"
