mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_multipart.py -x -q > gpurun_out/ch_test.log 2>&1; echo "rc=$?" >> gpurun_out/ch_test.log
MABD_LIB=paper_2603_08079_b200/libmabd.so timeout 120 python tools/exp_time.py 2 30 >> gpurun_out/ch_time.log 2>&1
MABD_LIB=paper_2603_08079_b200/libmabd.so timeout 120 python tools/exp_time.py 3 10 >> gpurun_out/ch_time.log 2>&1
