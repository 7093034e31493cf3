#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 BENCH_STREAM_PRIORITY=-5; do
    env $e timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/$e c2 /" >> gpurun_out/ab.jsonl
  done
done
