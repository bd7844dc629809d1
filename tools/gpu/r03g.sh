timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "axis_form or hyperdiffusion_parity or tile_ordered or laplacian_parity" > gpurun_out/r03g.log 2>&1; tail -2 gpurun_out/r03g.log
for i in 1 2; do
timeout 300 python tools/time_yt.py c5 2>&1 | grep "yt:" | tail -1
HV_LIB=/root/repo/ablate/prev/libhv_b200.so timeout 300 python tools/time_yt.py c5 2>&1 | grep "yt:" | tail -1
done
