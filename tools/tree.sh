mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_multipart.py tests/test_gpu_wrench.py tests/test_gpu_newton.py -x -q > gpurun_out/tr_test.log 2>&1; echo "rc=$?" >> gpurun_out/tr_test.log
timeout 300 python tools/exp_time.py 4 2 > gpurun_out/tr_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr_launches.csv python tools/exp_time.py 4 2 > gpurun_out/tr_ncu.log 2>&1
timeout 300 python bench.py --config 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg4.log 2>&1
