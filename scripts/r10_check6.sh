#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/check.jsonl
for w in c1 c3 c5; do
  SKB_DEBUG_SYNC=1 timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_${w}.err
done
SKB_DEBUG_SYNC=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_c2.err
