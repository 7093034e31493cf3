#!/bin/bash
mkdir -p gpurun_out/trace
SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c3 --warmup 5 --steps 20 --no-cpu-baseline > gpurun_out/trace/c3.json 2>&1
ls gpurun_out/trace
