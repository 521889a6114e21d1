#!/bin/bash
# re-entry check: GPU tests, smoke, default bench line, per-config lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in 1 3 4; do timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; done
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; for c in "" _cfg1 _cfg3 _cfg4; do tail -1 gpurun_out/bench$c.log | cut -c1-250; done
