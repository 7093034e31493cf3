#!/bin/bash
# CUPTI kernel timelines of C4 (exact) and C5 for critical-path reading
mkdir -p gpurun_out/trace
SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c4 --warmup 5 --steps 10 --no-cpu-baseline > gpurun_out/trace/c4.json 2>&1
SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c5 --warmup 5 --steps 10 --no-cpu-baseline > gpurun_out/trace/c5.json 2>&1
ls -la gpurun_out/trace
