#!/bin/bash
# TMA ring for mean / hot batches: parity of the variant tests, then same-box A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "variants" > gpurun_out/var_tests.log 2>&1; echo "rc=$?" >> gpurun_out/var_tests.log
CASES="base:SKB_X=0 hot:SKB_TMA_HOT=1 mean64:SKB_TMA_MEAN_MIN_D=64,SKB_TMA_HOT=1 mean48:SKB_TMA_MEAN_MIN_D=48 mean64c:SKB_TMA_MEAN_MIN_D=64" CONFIGS="c5 c4 c2" bash scripts/ab_env.sh
python scripts/ab_lib_show.py > gpurun_out/ab_show.txt
tail -2 gpurun_out/var_tests.log; cat gpurun_out/ab_show.txt
