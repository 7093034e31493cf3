#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/check.jsonl
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "growth or evict or vmm or restore or prefetch" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
for w in c3 c5 c1; do
  SKB_DEBUG_SYNC=1 timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_${w}.err
done
SKB_DEBUG_SYNC=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_c2.err
