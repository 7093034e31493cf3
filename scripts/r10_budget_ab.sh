#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 SKB_LF_BUDGET=160 SKB_LF_BUDGET=128 SKB_LF_BUDGET=96; do
    env $e timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/$e c4 /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
  done
done
for e in X=1 SKB_LF_BUDGET=128; do
  env $e timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/$e c5 /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
  env $e timeout 600 python bench.py --workload c3 --warmup 5 --steps 20 --no-cpu-baseline --c3-rows 40000000 | sed "s/^/$e c3 /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
mkdir -p gpurun_out/trace; SKB_LF_BUDGET=128 SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c4 --warmup 5 --steps 10 --no-cpu-baseline > /dev/null 2>&1
