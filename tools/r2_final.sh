#!/bin/bash
# round-2 closing evidence on one GPU: GPU tests, smoke, bench lines for configs 1-5, the default bench line, ncu launch
# lists (cfg2, cfg3, cfg4) and full captures of chain_kernel (cfg2) and the tree layer-0 UP kernel (cfg4)
mkdir -p gpurun_out
nvidia-smi > gpurun_out/f_nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench_default.log 2>&1
for c in 1 3 4 5; do
  st=100; [ $c = 5 ] && st=10; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/f_bench_cfg$c.log 2>&1
done
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/f_bench_cfg2.log 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/f_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_cfg2.csv $CMD > gpurun_out/f_ncu_l2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_cfg3.csv python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/f_ncu_l3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_cfg4.csv python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/f_ncu_l4.log 2>&1
python tools/exp_time.py 2 3 > gpurun_out/f_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/f_prof_chain python tools/exp_time.py 2 3 > gpurun_out/f_ncu_chain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tree_group_kernel -s 5 -c 1 -o gpurun_out/f_prof_tree python tools/exp_time.py 4 3 > gpurun_out/f_ncu_tree.log 2>&1
tail -2 gpurun_out/f_pytest_gpu.log; tail -1 gpurun_out/f_smoke.log
for f in default cfg1 cfg2 cfg3 cfg4 cfg5; do tail -1 gpurun_out/f_bench_$f.log | cut -c1-250; done
