#!/bin/bash
# C2 / C4 / C5 quick A/B line (run on the GPU box): ms per step of each
mkdir -p gpurun_out
TAG=${1:-x}
{
for i in 1 2; do
  timeout 600 python bench.py --warmup 5 --steps 50 --no-cpu-baseline | sed "s/^/c2 /"
  timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/c4 /"
  timeout 600 python bench.py --workload c5 --warmup 5 --steps 40 --no-cpu-baseline | sed "s/^/c5 /"
done
} > gpurun_out/ab_${TAG}.jsonl 2> gpurun_out/ab_${TAG}.err
