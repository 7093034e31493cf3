#!/bin/bash
mkdir -p gpurun_out/trace
SKB_DEBUG_SYNC=1 timeout 600 python bench.py --workload c3 --warmup 5 --steps 20 --no-cpu-baseline > gpurun_out/c3.json 2> gpurun_out/c3.err
SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/trace/c5.json 2> gpurun_out/trace/c5.err
