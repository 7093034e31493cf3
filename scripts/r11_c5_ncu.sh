#!/bin/bash
# ncu --set full of C5's fold+Adam launches (one per table) in a warm step
# NOTE: at C5 size the --set full replay fails (ncu backs up the multi-GB VMM arenas and the
# replayed launch fails); profiles/traffic_c5_r11.json (a 1-pass metric list) covers C5 instead.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fused_adam|k_fused_pool_stream" -s 20 -c 10 \
    -o gpurun_out/prof_c5_r11 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5_r11.log 2>&1
tail -2 gpurun_out/ncu_c5_r11.log
