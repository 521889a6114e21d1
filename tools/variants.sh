mkdir -p gpurun_out
for v in $VARIANTS; do
  if [ $v = default ]; then L=paper_2603_08079_b200/libmabd.so; else L=build_variants/lib_$v.so; fi
  MABD_LIB=$L timeout 120 python tools/exp_time.py 2 30 >> gpurun_out/variants.log 2>&1
done
