#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2 3; do
  for e in X=1; do
    env $e SKB_PROFILE_CALLS=1 timeout 600 python bench.py --workload c3 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/$e /" >> gpurun_out/ab.jsonl
    grep "fused_prepare\|backward_ex" gpurun_out/ab.err | tail -2 | sed "s/^/$e /" >> gpurun_out/ab_calls.txt
  done
done
