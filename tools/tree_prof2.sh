mkdir -p gpurun_out
MABD_LIB=build_variants/lib_tclk.so timeout 300 python tools/tclk.py 16 > gpurun_out/tclk.log 2>&1
