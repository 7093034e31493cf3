#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knobs.py tests/test_gpu_fullsize_oracle.py -m gpu -x -q -p no:cacheprovider -k "long or mega or hot or tile or tree or knob or graph or variants or c4 or C4" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/ab.jsonl
for i in 1 2; do
  for env in "X=1" "SKB_LF_EXCLUSIVE=0" "SKB_LF_STREAM_PACK=0"; do
    env $env timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/$env /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
  done
  for env in "X=1" "SKB_LF_STREAM_PACK=0"; do
    env $env timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/$env /" >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
  done
done
