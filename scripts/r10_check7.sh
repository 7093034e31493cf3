#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_oracle.py -m gpu -x -q -p no:cacheprovider -k "long or mega or hot or tile or tree or c4 or C4" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/check.jsonl
for w in c4 c5 c3; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_${w}.err
done
