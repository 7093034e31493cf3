#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 SKB_ADMIT_WAVES=4 SKB_ADMIT_WAVES=16; do
    env $e timeout 600 python bench.py --workload c3 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/$e c3 /" >> gpurun_out/ab.jsonl
  done
done
