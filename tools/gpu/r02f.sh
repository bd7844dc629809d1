timeout 300 python tools/time_yt.py c5 > gpurun_out/r02f_main.log 2>&1
HV_LIB=/root/repo/ablate/nopatch/libhv_b200.so timeout 300 python tools/time_yt.py c5 > gpurun_out/r02f_nopatch.log 2>&1
tail -6 gpurun_out/r02f_main.log gpurun_out/r02f_nopatch.log
timeout 600 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02f_main.csv python tools/time_yt.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
