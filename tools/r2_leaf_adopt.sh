#!/bin/bash
# leaf size 8 adopted: sparse-solver GPU tests, smoke and the config-5 bench line on the default library
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_frames.py tests/test_gpu_joints.py tests/test_gpu_limits.py tests/test_gpu_hinge5.py tests/test_gpu_strained.py tests/test_gpu_newton.py tests/test_gpu_line_gs.py tests/test_gpu_loop.py tests/test_gpu_graph.py tests/test_gpu_errors.py -q -p no:cacheprovider > gpurun_out/leaf8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/leaf8_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/leaf8_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/leaf8_smoke.log
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/leaf8_bench_cfg5.log 2>&1
tail -3 gpurun_out/leaf8_pytest.log; tail -1 gpurun_out/leaf8_smoke.log; tail -1 gpurun_out/leaf8_bench_cfg5.log | cut -c1-300
