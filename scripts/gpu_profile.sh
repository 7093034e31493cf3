#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list of the same
# command, and one `ncu --set full` capture of the fused-step kernels.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_fused_(adam_tma|pool_scatter|pool_staged|probe)|k_admission|DeviceRadixSortOnesweep" -s 20 -c 8 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${TAG}.log 2>&1
ls -la gpurun_out
