#!/bin/bash
# POTRF with the inverse by recursive doubling + MF_SG=2: full GPU suite and smoke on the default library,
# the cfg5 A/B against the previous POTRF (build_variants/lib_sg2.so), the cfg5 bench line and launch list
mkdir -p gpurun_out
for r in 1 2; do for v in build_variants/lib_sg2.so paper_2603_08079_b200/libmabd.so; do
  MABD_LIB=$v timeout 300 python tools/ab_sparse.py 5 >> gpurun_out/pf_ab.log 2>&1
done; done
cat gpurun_out/pf_ab.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/pf_bench_cfg5.log 2>&1
tail -1 gpurun_out/pf_bench_cfg5.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches_cfg5.csv python tools/ab_sparse.py 1 > gpurun_out/pf_ncu.log 2>&1; echo "ncu rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pf_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pf_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pf_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/pf_smoke.log
tail -2 gpurun_out/pf_pytest_gpu.log; tail -1 gpurun_out/pf_smoke.log
