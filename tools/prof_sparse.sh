# cfg5 sparse solver: plain timing, launch list (cold-cache, serialised), ncu --set full of the top kernels
mkdir -p gpurun_out
CMD="python tools/exp_time.py 5 1"
$CMD > gpurun_out/sp_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp_launches.csv $CMD > gpurun_out/sp_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mf_syrk_mma|mf_potrf|mf_ea|mf_small" -s 150 -c 8 -o gpurun_out/prof_sparse $CMD > gpurun_out/sp_ncu_full.log 2>&1
cat gpurun_out/sp_plain.log
