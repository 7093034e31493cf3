#!/bin/bash
mkdir -p gpurun_out/trace
SKB_LF_OVERLAP=0 SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c4 --warmup 5 --steps 10 --no-cpu-baseline > gpurun_out/trace/c4_nooverlap.json 2>&1
mv gpurun_out/trace/trace_c4.json gpurun_out/trace/trace_c4_nooverlap.json
