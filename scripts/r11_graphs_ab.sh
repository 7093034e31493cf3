#!/bin/bash
# CUDA-graph mode (every phase replayed as one graph) on the larger configs
CASES="eager:SKB_X=0 graphs:SKB_FUSED_GRAPHS=1" CONFIGS="c3 c5 c2" bash scripts/ab_env.sh
python scripts/ab_lib_show.py
tail -3 gpurun_out/ablib.err
