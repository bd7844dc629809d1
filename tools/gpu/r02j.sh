timeout 900 ncu --set full --import-source on --clock-control none -k regex:lap_plane_kernel --launch-skip 2 --launch-count 2 -o gpurun_out/r02j_yt python tools/time_yt.py c5 1 > gpurun_out/r02j.log 2>&1; echo ncu rc=$?
ls -la gpurun_out/
