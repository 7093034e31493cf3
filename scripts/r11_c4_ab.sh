#!/bin/bash
# C4: main fold co-running with the long fold (occupancy) — variant / grid A/B
CASES="base:SKB_X=0 r2:SKB_ADAM_VARIANT=1 r1b5:SKB_ADAM_VARIANT=2 g100:SKB_LF_GRID=100 g74:SKB_LF_GRID=74 r2g100:SKB_ADAM_VARIANT=1,SKB_LF_GRID=100" CONFIGS="c4" bash scripts/ab_env.sh
python scripts/ab_lib_show.py
