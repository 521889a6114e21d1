#!/bin/bash
# A/B timing of library variants: bash tools/ab2.sh lib_a lib_b ... (names of build_exp/<name>.so)
mkdir -p gpurun_out
for i in 1 2; do
for v in "$@"; do
  L=build_exp/$v.so
  r2=$(MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; [print(round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]")
  r3=$(MABD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --config 3 --steps 20 2>&1 | python -c "import json,sys; [print(round(json.loads(l)['ms_per_step']*1e3,1)) for l in sys.stdin if l.startswith('{')]")
  echo "$v cfg2 $r2 us  cfg3 $r3 us"
done; done
