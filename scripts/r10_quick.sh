#!/bin/bash
# quick: hot-id parity tests + C4/C5 lines + VMM call costs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "long or mega or hot or tile or variants or tree" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
: > gpurun_out/quick.jsonl
for w in c4 c5; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/quick.jsonl 2> gpurun_out/quick_${w}.err
done
SKB_LF_PACK=0 timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline >> gpurun_out/quick.jsonl 2>> gpurun_out/quick_c4.err
timeout 120 python scripts/vmm_timing.py > gpurun_out/vmm_timing.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4q.csv \
    -k regex:"k_pack_rows|k_long_fold|k_fused_adam|k_fused_tile" python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
