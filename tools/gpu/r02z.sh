timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02z.log 2>&1
grep -E "^FAILED|Error" gpurun_out/r02z.log | head -20; tail -2 gpurun_out/r02z.log
for c in c3; do timeout 300 python tools/time_secondary.py $c 20 2>&1 | tail -1; done
timeout 300 python tools/time_yt.py c5 2>&1 | grep -v Warn | tail -3
timeout 300 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem --clock-control none --csv --log-file gpurun_out/r02z_c3.csv python tools/time_secondary.py c3 1 > /dev/null 2>&1; echo ncu rc=$?
