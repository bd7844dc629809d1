for i in 1 2; do
timeout 300 python tools/time_yt.py c5 2>&1 | grep "yt:" | tail -1
HV_LIB=/root/repo/ablate/prev/libhv_b200.so timeout 300 python tools/time_yt.py c5 2>&1 | grep "yt:" | tail -1
done
