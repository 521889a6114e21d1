#!/bin/bash
# A/B of the nested-dissection leaf size (MF_LEAF_P) and the small-front limit (MF_SMALL_F) on config 5
mkdir -p gpurun_out; rm -f gpurun_out/leaf_ab.log
for r in 1 2; do for v in paper_2603_08079_b200/libmabd.so $VARS; do
  MABD_LIB=$v timeout 200 python tools/ab_sparse.py 5 2>&1 | tail -1 >> gpurun_out/leaf_ab.log
done; done
cat gpurun_out/leaf_ab.log
