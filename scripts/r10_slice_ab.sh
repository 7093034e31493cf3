#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_knobs.py -m gpu -x -q -p no:cacheprovider > gpurun_out/knob_tests.log 2>&1; echo "rc=$?" >> gpurun_out/knob_tests.log
: > gpurun_out/ab.jsonl
for i in 1 2; do
for sl in 0 512 768 1536 2048; do
  SKB_TMA_SLICE=$sl timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline | sed "s/^/$sl /" >> gpurun_out/ab.jsonl 2>/dev/null
done
done
