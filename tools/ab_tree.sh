#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do for v in $VARS; do
  MABD_LIB=build_variants/lib_$v.so timeout 200 python tools/ab_tree.py >> gpurun_out/ab_tree.log 2>&1
done; done
cat gpurun_out/ab_tree.log
