for c in c2 c3; do HV_DISABLE_TILES=1 timeout 300 python tools/time_secondary.py $c 20 2>&1 | tail -1; done
for c in c2; do HV_KERNEL=line timeout 300 python tools/time_secondary.py $c 20 2>&1 | tail -1; done
