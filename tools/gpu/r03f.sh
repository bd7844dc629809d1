timeout 600 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "c4 or euler or rhs" > gpurun_out/r03f.log 2>&1; tail -2 gpurun_out/r03f.log
for i in 1 2; do timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1; HV_EULER_NPT=1 timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1; done
timeout 300 ncu --kernel-name regex:"euler" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03f.csv python tools/time_secondary.py c4 1 > /dev/null 2>&1; echo ncu rc=$?
