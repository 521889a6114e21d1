#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, per-config bench lines, ncu launch list + full capture.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in 1 3 4; do timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; done
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5.log 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/prof_chain $CMD > gpurun_out/ncu_full.log 2>&1
echo done
# the tree path (config 4): launch list and one full capture of the layer-0 UP kernel
TCMD="python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr_launches.csv $TCMD > gpurun_out/tr_ncu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tree_group_kernel -s 5 -c 1 -o gpurun_out/prof_tree $TCMD > gpurun_out/tr_ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
echo done2
