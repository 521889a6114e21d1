mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_multipart.py -x -q > gpurun_out/ch_test.log 2>&1; echo "rc=$?" >> gpurun_out/ch_test.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --config 3 --steps 20 --warmup 3 > gpurun_out/bench_quick3.log 2>&1
