#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_distributed.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "dist or fold or grad or partition or a2a or restore" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 SKB_POOL_BY_INDEX_STREAM=0 SKB_FOLD_ONLY_R=1; do
    env $e BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 2>>gpurun_out/ab.err | sed "s/^/$e n2 /" >> gpurun_out/ab.jsonl
  done
done
