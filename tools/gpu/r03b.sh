timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4.py -q -p no:cacheprovider > gpurun_out/r03b.log 2>&1
grep -E "^FAILED|Error" gpurun_out/r03b.log | head -20; tail -2 gpurun_out/r03b.log
for i in 1 2; do timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1; HV_YT7=1 timeout 300 python tools/time_secondary.py c4 2>&1 | tail -1; done
