#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "tree_fold" > gpurun_out/tree.log 2>&1; echo "rc=$?" >> gpurun_out/tree.log
SKB_DEBUG_SYNC=1 timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --csv --log-file gpurun_out/randacc.csv python scripts/random_access_bench.py > gpurun_out/randacc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r10.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_fused_(adam_tma|pool_scatter|pool_staged|probe)|k_admission|DeviceRadixSortOnesweep" -s 20 -c 8 \
    -o gpurun_out/prof_r10 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r10.log 2>&1
ls -la gpurun_out
