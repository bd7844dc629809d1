timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tile_ordered or hyperdiffusion_parity or laplacian_parity" > gpurun_out/r02d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02d_pytest.log
tail -3 gpurun_out/r02d_pytest.log
timeout 600 python tools/time_yt.py c5 > gpurun_out/r02d_time.log 2>&1
timeout 300 python tools/time_yt.py c3 >> gpurun_out/r02d_time.log 2>&1
grep -v Warn gpurun_out/r02d_time.log
timeout 600 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02d_launches.csv python tools/time_yt.py c5 1 > gpurun_out/r02d_ncu.log 2>&1; echo ncu rc=$?
