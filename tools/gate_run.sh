# panel-POTRF A/B on cfg5: launch-list totals per variant, then the bench line of the default
mkdir -p gpurun_out
CMD="python tools/exp_time.py 5 1"
for v in reg block; do
  if [ $v = block ]; then export MABD_SPARSE_POTRF_BLOCK=1; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:mf_potrf -c 141 $CMD 2>/dev/null | grep potrf | awk -F'","' -v V=$v '{s+=$NF; n++} END {print V, "potrf launches", n, "total us", s/1000, "mean", s/n/1000}'
done
unset MABD_SPARSE_POTRF_BLOCK
python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -1
b() { timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['frac'])"; }
b reg
MABD_SPARSE_POTRF_BLOCK=1 b block
