#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "pool or onehot or variants or fused" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/check.jsonl
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_c2.err
for w in c5 c1; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_${w}.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5q.csv \
    -k regex:"k_fused_pool|k_fused_adam" python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
