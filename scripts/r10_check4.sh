#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/check.jsonl
for w in c5 c1 c3; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_${w}.err
done
timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline --fold tree >> gpurun_out/check.jsonl 2>> gpurun_out/check_c5.err
for i in 1 2; do
timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2>> gpurun_out/check_c4.err
SKB_LF_EXCLUSIVE=1 timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2>> gpurun_out/check_c4.err
done
