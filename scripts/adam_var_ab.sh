#!/bin/bash
# C5 fold+Adam kernel variants: per-table kernel times from a CUPTI trace
# (scripts/adam_var_show.py reads gpurun_out/av/*)
mkdir -p gpurun_out/av
for v in ${VARS:-0 1 2 3 4 7 9}; do
  mkdir -p gpurun_out/av/v$v
  SKB_ADAM_VARIANT=$v SKB_TRACE=gpurun_out/av/v$v timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 \
    --no-cpu-baseline > gpurun_out/av/v$v.jsonl 2> gpurun_out/av/v$v.err
done
