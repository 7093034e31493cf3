#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
: > gpurun_out/configs_r10.jsonl
for w in c1 c3 c4 c5; do
  timeout 600 python bench.py --workload $w --warmup 5 $([ $w = c1 ] || echo --steps 20) >> gpurun_out/configs_r10.jsonl 2> gpurun_out/cfg_${w}.err
done
for w in c3 c4 c5; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --fold tree >> gpurun_out/configs_r10.jsonl 2> gpurun_out/cfg_${w}_tree.err
done
BENCH_SHARED_GPU=1 SKB_DEBUG_SYNC=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err
timeout 300 python ops_bench.py > gpurun_out/ops_r10.txt 2>&1
timeout 300 python ops_bench.py --rows > gpurun_out/ops_rows_r10.txt 2>&1
ls -la gpurun_out
