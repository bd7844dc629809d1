timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4.py tests/test_parallel.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02l.csv python tools/time_yt.py c5 1 > gpurun_out/r02l.log 2>&1; echo ncu rc=$?
timeout 300 python tools/time_yt.py c5 2>&1 | grep -v Warn
timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1
