#!/bin/bash
# grouped triangular-solve launches (MF_SG): sparse GPU tests on the default library, then the cfg5 A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_frames.py tests/test_gpu_joints.py tests/test_gpu_limits.py tests/test_gpu_hinge5.py tests/test_gpu_strained.py tests/test_gpu_newton.py -q -x -p no:cacheprovider > gpurun_out/sg_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sg_pytest.log
for r in 1 2; do for v in build_variants/lib_zfull.so build_variants/lib_sg1.so build_variants/lib_sg2.so paper_2603_08079_b200/libmabd.so build_variants/lib_sg8.so; do
  MABD_LIB=$v timeout 300 python tools/ab_sparse.py 5 >> gpurun_out/sg_ab.log 2>&1
done; done
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/sg_bench_cfg5.log 2>&1
tail -3 gpurun_out/sg_pytest.log; cat gpurun_out/sg_ab.log; tail -1 gpurun_out/sg_bench_cfg5.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sg_launches_cfg5.csv python tools/ab_sparse.py 1 > gpurun_out/sg_ncu.log 2>&1; echo "ncu rc=$?"
