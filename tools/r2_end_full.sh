#!/bin/bash
# full GPU suite on the final library (the tests the leaf-size run did not include come first)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_longrun.py tests/test_gpu_polarfree.py tests/test_gpu_wrench.py tests/test_gpu_single_body.py tests/test_gpu_exchange.py tests/test_gpu_multipart.py tests/test_gpu_chain.py tests/test_gpu_tree.py -m gpu -q -p no:cacheprovider > gpurun_out/end2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/end2_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/end2_bench_default.log 2>&1
tail -3 gpurun_out/end2_pytest_gpu.log; tail -1 gpurun_out/end2_bench_default.log | cut -c1-300
