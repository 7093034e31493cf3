#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"k_write_rows_if_clear|k_check_rows" -c 6 -o gpurun_out/prof_rows python ops_bench.py > gpurun_out/ncu_rows.log 2>&1
tail -2 gpurun_out/ncu_rows.log
