#!/bin/bash
# round-2 closing run on the final library: GPU tests, smoke, default bench line, bench lines of configs 1-5,
# cfg2 launch list and a full capture of chain_kernel
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g_smoke.log
timeout 900 python bench.py > gpurun_out/g_bench_default.log 2>&1
for c in 1 3 4 5; do
  st=100; [ $c = 5 ] && st=10; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/g_bench_cfg$c.log 2>&1
done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/g_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_cfg2.csv $CMD > gpurun_out/g_ncu_l2.log 2>&1
python tools/exp_time.py 2 3 > gpurun_out/g_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/g_prof_chain python tools/exp_time.py 2 3 > gpurun_out/g_ncu_chain.log 2>&1
tail -2 gpurun_out/g_pytest_gpu.log; tail -1 gpurun_out/g_smoke.log
for f in default cfg1 cfg3 cfg4 cfg5; do tail -1 gpurun_out/g_bench_$f.log | cut -c1-250; done
