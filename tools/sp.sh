mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q -k "not full_size" > gpurun_out/sp_test.log 2>&1; echo "rc=$?" >> gpurun_out/sp_test.log
timeout 300 python tools/sp_refine.py 64 5 > gpurun_out/sp_refine.log 2>&1
timeout 900 python tools/sp_refine.py 512 1 >> gpurun_out/sp_refine.log 2>&1
