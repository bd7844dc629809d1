for L in paper_2311_11425_b200/libhv_b200.so ablate/nopatch/libhv_b200.so; do
HV_LIB=$L timeout 600 ncu --kernel-name regex:"lap_plane|slot_fixup" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02e_$(basename $(dirname $L)).csv python tools/time_yt.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
done
