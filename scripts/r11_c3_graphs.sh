#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ablib.jsonl
for i in 1 2 3 4; do
  for case in eager:SKB_X=0 graphs:SKB_FUSED_GRAPHS=1; do
    name=${case%%:*}; envs=${case#*:}
    env $envs timeout 600 python bench.py --workload c3 --warmup 5 --steps 40 --no-cpu-baseline | sed "s/^/$name c3 /" >> gpurun_out/ablib.jsonl
  done
done 2> gpurun_out/ablib.err
python scripts/ab_lib_show.py
