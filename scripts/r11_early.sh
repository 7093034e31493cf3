#!/bin/bash
# early tile forward: parity (tile tests, knob subprocesses), then same-box C4 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "tile or early or knob" > gpurun_out/early_tests.log 2>&1; echo "rc=$?" >> gpurun_out/early_tests.log
tail -3 gpurun_out/early_tests.log
: > gpurun_out/ablib.jsonl
for i in 1 2; do
  for e in 1 0; do
    SKB_TILE_EARLY=$e timeout 600 python bench.py --workload c4 --warmup 5 --steps 30 --no-cpu-baseline 2>>gpurun_out/ablib.err | sed "s/^/early$e c4 /" >> gpurun_out/ablib.jsonl
    SKB_TILE_EARLY=$e timeout 600 python bench.py --workload c4 --warmup 5 --steps 30 --no-cpu-baseline --fold tree 2>>gpurun_out/ablib.err | sed "s/^/early$e c4tree /" >> gpurun_out/ablib.jsonl
  done
done
python scripts/ab_lib_show.py
mkdir -p gpurun_out/trace
SKB_TRACE=gpurun_out/trace timeout 600 python bench.py --workload c4 --warmup 5 --steps 10 --no-cpu-baseline > gpurun_out/trace/c4e.json 2>&1
