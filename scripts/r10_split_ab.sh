#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knobs.py -m gpu -x -q -p no:cacheprovider -k "long or mega or hot or tile or knob or variants" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for e in X=1 SKB_LF_SPLIT=0; do
    env $e timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/$e c4 /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
  done
done
timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/c5 /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
mkdir -p gpurun_out/trace; SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c4 --warmup 5 --steps 10 --no-cpu-baseline > /dev/null 2>&1
