mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q -k "not full_size" > gpurun_out/sp_test.log 2>&1; echo "rc=$?" >> gpurun_out/sp_test.log
timeout 300 python tools/exp_time.py 5 3 > gpurun_out/sp_time.log 2>&1
timeout 300 python tools/exp_time.py 5 1 > gpurun_out/sp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp_launches.csv python tools/exp_time.py 5 1 > gpurun_out/sp_ncu.log 2>&1
