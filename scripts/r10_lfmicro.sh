#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/lfmicro.txt
for n in 387000 774000 1548000; do
  LF_N=$n LF_D=64 LF_HOT=1.0 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__cycles_elapsed.avg.per_second --clock-control none -k regex:"k_long_fold|k_pack_rows" --csv python scripts/longfold_bench.py 2>/dev/null | grep -E "k_long_fold|k_pack_rows" | tail -4 | sed "s/^/n=$n /" >> gpurun_out/lfmicro.txt
done
