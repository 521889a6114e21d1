mkdir -p gpurun_out
CMD="python tools/exp_time.py 5 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mf_potrf|mf_small|mf_syrk" -s 200 -c 6 -o gpurun_out/prof_sparse $CMD > gpurun_out/ncu_full.log 2>&1
