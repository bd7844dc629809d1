timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02o.log 2>&1
grep -E "^FAILED|Error" gpurun_out/r02o.log | head -30; tail -2 gpurun_out/r02o.log
