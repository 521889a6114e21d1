mkdir -p gpurun_out
CMD="python tools/exp_time.py 4 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 19 -c 19 -o gpurun_out/prof_tree2 $CMD > gpurun_out/ncu_full.log 2>&1
