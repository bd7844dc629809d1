set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tile_ordered or hyperdiffusion_parity or laplacian_parity" > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
tail -3 gpurun_out/r02b_pytest.log
timeout 600 python tools/time_yt.py c5 > gpurun_out/r02b_time.log 2>&1
timeout 300 python tools/time_yt.py c2 >> gpurun_out/r02b_time.log 2>&1
timeout 300 python tools/time_yt.py c3 >> gpurun_out/r02b_time.log 2>&1
cat gpurun_out/r02b_time.log | grep -v Warn
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02b_launches.csv python tools/time_yt.py c5 > /dev/null 2>&1; echo ncu rc=$?
