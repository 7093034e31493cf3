#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knobs.py tests/test_gpu_fullsize_oracle.py -m gpu -x -q -p no:cacheprovider -k "long or mega or hot or tile or tree or knob or graph or variants or c4 or C4 or c5 or C5" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/ab.jsonl
for w in c4 c5 c3 c4; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
mkdir -p gpurun_out/trace; SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c4 --warmup 5 --steps 10 --no-cpu-baseline > /dev/null 2>&1
