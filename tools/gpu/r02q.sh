timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tile_ordered or hyperdiffusion_parity" > gpurun_out/r02q_t.log 2>&1; tail -3 gpurun_out/r02q_t.log
timeout 300 python tools/time_yt.py c5 > gpurun_out/r02q.log 2>&1; grep -v Warn gpurun_out/r02q.log | tail -6
timeout 300 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02q.csv python tools/time_yt.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
