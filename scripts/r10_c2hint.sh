#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2 3; do
  SKB_DEBUG_SYNC=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/c2 /" >> gpurun_out/ab.jsonl
done
