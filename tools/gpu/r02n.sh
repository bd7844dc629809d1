timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4.py -q -p no:cacheprovider > gpurun_out/r02n.log 2>&1
grep -E "^FAILED|Error|assert " gpurun_out/r02n.log | head -30; tail -3 gpurun_out/r02n.log
