#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_part_" -c 8 -o gpurun_out/prof_part python ops_bench.py > gpurun_out/ncu_part.log 2>&1
tail -3 gpurun_out/ncu_part.log
