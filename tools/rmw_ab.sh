mkdir -p gpurun_out
for v in prev cur; do MABD_LIB=build_variants/lib_$v.so timeout 300 python tools/exp_time.py 4 20 2>&1 | grep -v "solver stats"; MABD_LIB=build_variants/lib_$v.so timeout 300 python tools/exp_time.py 5 3 2>&1 | grep -v "solver stats"; done > gpurun_out/rmw.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:"sparse_predict|sparse_update" --csv --log-file gpurun_out/k14b.csv python tools/k14.py > gpurun_out/k14b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_sparse.py tests/test_gpu_newton.py tests/test_gpu_wrench.py -x -q > gpurun_out/rmw_test.log 2>&1; tail -2 gpurun_out/rmw_test.log >> gpurun_out/rmw.log
