#!/bin/bash
# per-rank step time of config 2's strong split (4096/W chains per rank, no collective), one GPU
mkdir -p gpurun_out
timeout 600 python tools/cfg2_shard_probe.py 100 > gpurun_out/shard_probe.log 2>&1; echo "rc=$?" >> gpurun_out/shard_probe.log
cat gpurun_out/shard_probe.log
