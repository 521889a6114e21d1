#!/bin/bash
# A/B of chain-kernel variants (build_variants/lib_<v>.so): device time per step of cfg2 (100-step episodes) and cfg3
mkdir -p gpurun_out
VARS=${VARS:-"base va vad"}
for i in 1 2; do
for v in $VARS; do
  L=build_variants/lib_$v.so
  echo "== $v" >> gpurun_out/ab_r2c.log
  MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; [print('cfg2', round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/ab_r2c.log
  MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --config 3 --steps 20 2>&1 | python -c "import json,sys; [print('cfg3', round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/ab_r2c.log
done; done
cat gpurun_out/ab_r2c.log
