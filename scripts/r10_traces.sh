#!/bin/bash
# CUPTI kernel timelines (torch.profiler) of a few steps after each timed region
mkdir -p gpurun_out/trace
export SKB_TRACE=gpurun_out/trace
timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/trace/c2.json 2> gpurun_out/trace/c2.err
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/trace/c5.json 2> gpurun_out/trace/c5.err
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/trace/c4.json 2> gpurun_out/trace/c4.err
BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/trace/n2.json 2> gpurun_out/trace/n2.err
ls -la gpurun_out/trace
