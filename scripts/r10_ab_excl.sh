#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2; do
for w in c5 c3 c4; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline --c3-rows 40000000 >> gpurun_out/ab.jsonl 2>/dev/null
  SKB_LF_EXCLUSIVE=1 timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline --c3-rows 40000000 >> gpurun_out/ab.jsonl 2>/dev/null
done
done
