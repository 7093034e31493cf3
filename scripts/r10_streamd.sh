#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 SKB_POOL_STREAM_MIN_D=32 SKB_POOL_STREAM_MIN_D=16 SKB_POOL_STREAM_MIN_D=8; do
    env $e timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/$e c5 /" >> gpurun_out/ab.jsonl
  done
done
SKB_POOL_STREAM_MIN_D=8 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "pool or onehot or mean or fused_vs or variants" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
