mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_multipart.py tests/test_gpu_tree.py -x -q > gpurun_out/ch_test.log 2>&1; echo "rc=$?" >> gpurun_out/ch_test.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
