#!/bin/bash
# host-side profile of the C5 step loop (cProfile; the timed steps only are
# read back with scripts/prof_show.py)
mkdir -p gpurun_out
timeout 900 python -m cProfile -o gpurun_out/c5.prof bench.py --workload c5 --warmup 5 --steps 40 --no-cpu-baseline > gpurun_out/c5prof.jsonl 2> gpurun_out/c5prof.err
