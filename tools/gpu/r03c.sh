timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tile_ordered or hyperdiffusion_parity or segments" > gpurun_out/r03c_t.log 2>&1; tail -2 gpurun_out/r03c_t.log
for i in 1 2; do timeout 300 python tools/time_yt.py c5 2>&1 | grep -v Warn | tail -3; done
timeout 300 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r03c.csv python tools/time_yt.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
