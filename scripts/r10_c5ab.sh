#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 SKB_LF_CARVEOUT=-1 SKB_LF_STREAM_PACK=0; do
    env $e timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/$e c5 /" >> gpurun_out/ab.jsonl
  done
done
