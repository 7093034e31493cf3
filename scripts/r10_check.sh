#!/bin/bash
# parity after a kernel change + the config lines it targets
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
: > gpurun_out/check.jsonl
for w in c4 c5 c1; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_${w}.err
done
BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 >> gpurun_out/check.jsonl 2> gpurun_out/check_n2.err
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/check.jsonl 2> gpurun_out/check_c2.err
