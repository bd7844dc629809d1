timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4.py -q -p no:cacheprovider > gpurun_out/r03a.log 2>&1
grep -E "^FAILED|Error" gpurun_out/r03a.log | head -20; tail -2 gpurun_out/r03a.log
timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1
HV_YT=0 timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1
timeout 300 ncu --kernel-name regex:"lap_plane|slot_fixup|euler" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r03a.csv python tools/time_secondary.py c4 1 > /dev/null 2>&1; echo ncu rc=$?
