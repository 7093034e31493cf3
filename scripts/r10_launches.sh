#!/bin/bash
# launch lists (serialized per-kernel times) of the shared-GPU N=2 step, C5 and C4
mkdir -p gpurun_out
BENCH_SHARED_GPU=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n2_r10.csv \
    python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/n2_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r10.csv \
    python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r10.csv \
    python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_r10.csv \
    python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c1_ncu.log 2>&1
ls -la gpurun_out
