#!/bin/bash
# A/B of a C2 knob: default vs env override, interleaved
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2 3; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline >> gpurun_out/ab.jsonl 2>/dev/null
  SKB_TMA_WHOLE_WAVES=0 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline >> gpurun_out/ab.jsonl 2>/dev/null
done
