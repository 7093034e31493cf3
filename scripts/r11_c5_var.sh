#!/bin/bash
# C5: fold+Adam register shapes per table width (same box)
CASES="base:SKB_X=0 n1:SKB_C5_VARIANTS=8:1:-1/16:1:-1 n2:SKB_C5_VARIANTS=8:2:-1/16:2:-1 n1w:SKB_C5_VARIANTS=8:1:-1/16:1:-1/32:1:-1 w2:SKB_C5_VARIANTS=64:2:-1/128:2:-1 w1:SKB_C5_VARIANTS=64:1:-1/128:1:-1" CONFIGS="c5" bash scripts/ab_env.sh
python scripts/ab_lib_show.py
tail -3 gpurun_out/ablib.err
