#!/bin/bash
# A/B of library variants: VARS="a b c" → build_variants/lib_<v>.so, alternated 3 times
mkdir -p gpurun_out
for i in 1 2 3; do for v in $VARS; do
  MABD_LIB=build_variants/lib_$v.so timeout 200 python tools/ab_time.py >> gpurun_out/ab_r2d.log 2>&1
done; done
cat gpurun_out/ab_r2d.log
