#!/bin/bash
# same-box A/B of library builds: SKB_LIB_PATH=abso/lib_<v>.so for each v,
# interleaved, C2 / C4 / C5 (ms per step lines -> gpurun_out/ablib.jsonl)
mkdir -p gpurun_out
: > gpurun_out/ablib.jsonl
for i in 1 2; do
  for v in $VARIANTS; do
    export SKB_LIB_PATH=abso/lib_$v.so
    timeout 600 python bench.py --warmup 5 --steps 50 --no-cpu-baseline | sed "s/^/$v c2 /" >> gpurun_out/ablib.jsonl
    [ -n "$NO_C4" ] || timeout 600 python bench.py --workload c4 --warmup 5 --steps 20 --no-cpu-baseline | sed "s/^/$v c4 /" >> gpurun_out/ablib.jsonl
    timeout 600 python bench.py --workload c5 --warmup 5 --steps 40 --no-cpu-baseline | sed "s/^/$v c5 /" >> gpurun_out/ablib.jsonl
  done
done 2> gpurun_out/ablib.err
