#!/bin/bash
# C5: TMA ring shapes on the wide tables only (per-table override)
CASES="base:SKB_X=0 t128v8:SKB_C5_VARIANTS=128:8:-1 t128v7:SKB_C5_VARIANTS=128:7:-1 t128v5:SKB_C5_VARIANTS=128:5:-1 t128v4:SKB_C5_VARIANTS=128:4:-1 t64v6:SKB_C5_VARIANTS=64:6:-1 t64v4:SKB_C5_VARIANTS=64:4:-1" CONFIGS="c5" bash scripts/ab_env.sh
python scripts/ab_lib_show.py
tail -3 gpurun_out/ablib.err
