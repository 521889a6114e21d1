mkdir -p gpurun_out
CMD="python tools/exp_time.py 2 3"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/prof_chain_v4 $CMD > gpurun_out/ncu_full.log 2>&1
