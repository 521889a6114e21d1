#!/bin/bash
# round-2 re-entry: GPU tests, default bench line, chain_kernel full capture
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/c_bench_cfg2.log 2>&1
python tools/exp_time.py 2 3 > gpurun_out/c_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/c_prof_chain python tools/exp_time.py 2 3 > gpurun_out/c_ncu_full.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest_gpu.log
tail -1 gpurun_out/c_bench_cfg2.log; tail -3 gpurun_out/c_pytest_gpu.log
