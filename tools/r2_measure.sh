#!/bin/bash
# round-2 evidence: fp64 peak, bench lines for configs 1-5, ncu captures of the sparse factorization kernels
mkdir -p gpurun_out
./build_exp/fp64_peak > gpurun_out/r2_fp64_peak.log 2>&1
for c in 1 3 4 5; do
  st=100; [ $c = 5 ] && st=10; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --e2e-steps 2 > gpurun_out/r2_bench_cfg$c.log 2>&1
done
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/r2_bench_cfg2.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --rotation length_preserving > gpurun_out/r2_bench_cfg2_lp.log 2>&1
timeout 600 python tools/exp_time.py 5 1 > gpurun_out/r2_sp_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"mf_syrk|mf_potrf|mf_ea|mf_trsm" -s 40 -c 4 -o gpurun_out/r2_prof_sparse python tools/exp_time.py 5 1 > gpurun_out/r2_ncu_sparse.log 2>&1
cat gpurun_out/r2_fp64_peak.log; for c in 1 2 3 4 5; do tail -1 gpurun_out/r2_bench_cfg$c.log | cut -c1-300; done
