mkdir -p gpurun_out
for i in 1 2; do
for v in prev cur; do
  L=build_variants/lib_$v.so
  echo "== $v" >> gpurun_out/ab.log
  MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; [print('bench', round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/ab.log
  MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --config 3 --steps 20 2>&1 | python -c "import json,sys; [print('bench3', round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/ab.log
done; done
