#!/bin/bash
# chain-kernel evidence on one GPU: phase split (clock build), bench line, ncu full capture of chain_kernel
mkdir -p gpurun_out
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_cfg2.log 2>&1
MABD_LIB=build_exp/lib_clk.so python tools/exp_time.py 2 20 > gpurun_out/r2_clk.log 2>&1
python tools/exp_time.py 2 3 > gpurun_out/r2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/r2_prof_chain python tools/exp_time.py 2 3 > gpurun_out/r2_ncu_full.log 2>&1
tail -1 gpurun_out/r2_bench_cfg2.log; cat gpurun_out/r2_clk.log
