mkdir -p gpurun_out
for v in prev cur prev cur; do
  echo "== $v" >> gpurun_out/ab5.log
  MABD_LIB=build_variants/lib_$v.so timeout 300 python tools/exp_time.py 5 3 2>&1 | grep -v "solver stats" >> gpurun_out/ab5.log
done
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_longrun.py -x -q -k "sparse or cfg5 or ring or net" > gpurun_out/sp_test.log 2>&1; tail -2 gpurun_out/sp_test.log >> gpurun_out/ab5.log
