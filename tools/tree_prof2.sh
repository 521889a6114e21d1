mkdir -p gpurun_out
MABD_LIB=build_variants/lib_tclk.so timeout 300 python tools/tclk.py 16 > gpurun_out/tclk.log 2>&1
timeout 300 python tools/exp_time.py 4 20 > gpurun_out/tr_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/tr_launches_warm.csv python tools/exp_time.py 4 2 > gpurun_out/tr_ncu.log 2>&1
