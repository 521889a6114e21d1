#!/bin/bash
# A/B of library variants on cfg2 / cfg3 (bench.py device time), then the chain parity tests on the last variant
mkdir -p gpurun_out; : > gpurun_out/ab3.log
VARS="$@"
for i in 1 2; do
for v in $VARS; do
  L=build_variants/lib_$v.so
  a=$(MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; [print(round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]")
  b=$(MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --config 3 --steps 20 2>&1 | python -c "import json,sys; [print(round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]")
  echo "$v cfg2 $a cfg3 $b" >> gpurun_out/ab3.log
done; done
last=${@: -1}
MABD_LIB=build_variants/lib_$last.so timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_strained.py tests/test_gpu_longrun.py tests/test_gpu_frames.py -m gpu -x -q > gpurun_out/ab3_tests.log 2>&1
tail -2 gpurun_out/ab3_tests.log >> gpurun_out/ab3.log
cat gpurun_out/ab3.log
