#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "growth or evict or vmm or restore or prefetch or checkpoint" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/ab.jsonl
for i in 1 2 3; do
  timeout 600 python bench.py --workload c3 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/c3 /" >> gpurun_out/ab.jsonl
done
timeout 600 python bench.py --workload c5 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/c5 /" >> gpurun_out/ab.jsonl
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/c2 /" >> gpurun_out/ab.jsonl
timeout 600 python bench.py --workload c1 --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/ab.err | sed "s/^/c1 /" >> gpurun_out/ab.jsonl
