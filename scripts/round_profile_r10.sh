#!/bin/bash
# Everything profiles/ needs for round r10 (run on the GPU box via gpurun).
TAG=${1:-r10}
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
: > gpurun_out/configs_${TAG}.jsonl
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --warmup 5 $([ $w = c1 ] || echo --steps 20) >> gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/cfg_${w}.err
done
for w in c3 c4 c5; do
  timeout 900 python bench.py --workload $w --warmup 5 --steps 20 --fold tree --no-cpu-baseline >> gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/cfg_${w}_tree.err
done
BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_shared_${TAG}.json 2> gpurun_out/bench_n2_shared_${TAG}.err
timeout 300 python ops_bench.py > gpurun_out/ops_${TAG}.txt 2>&1
timeout 300 python ops_bench.py --rows > gpurun_out/ops_rows_${TAG}.txt 2>&1
# launch list of the headline command, and per-step DRAM traffic of every config's timed region
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for w in c2 c4 c5 c3; do
  timeout 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/traffic_${w}_${TAG}.csv \
      python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline $([ $w = c3 ] && echo --c3-rows 20000000) > gpurun_out/traffic_${w}.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"k_fused_(adam_tma|pool_scatter|pool_staged|probe)|k_admission|DeviceRadixSortOnesweep" -s 20 -c 8 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${TAG}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"k_long_fold|k_pack_rows|k_fused_pool_stream|k_fused_adam" -s 6 -c 6 \
    -o gpurun_out/prof_c4c5_${TAG} python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4_${TAG}.log 2>&1
ls -la gpurun_out
