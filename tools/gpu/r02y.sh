timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "segments or tile_ordered or hyperdiffusion_parity" > gpurun_out/r02y.log 2>&1; grep -E "^FAILED|Error|assert " gpurun_out/r02y.log | head; tail -2 gpurun_out/r02y.log
for s in 0 1 2 4; do HV_SEG=$s timeout 300 python tools/time_secondary.py c2 20 2>&1 | tail -1; done
for s in 0 5; do HV_SEG=$s timeout 300 python tools/time_secondary.py c3 20 2>&1 | tail -1; done
