#!/bin/bash
# same-box A/B of environment knobs: CASES="name:VAR=val,VAR2=val name2:..." ;
# CONFIGS="c2 c4 c5" -> gpurun_out/ablib.jsonl (read with scripts/ab_lib_show.py)
mkdir -p gpurun_out
: > gpurun_out/ablib.jsonl
for i in 1 2; do
  for case in $CASES; do
    name=${case%%:*}; envs=${case#*:}
    for c in ${CONFIGS:-c2 c4 c5}; do
      args="--workload $c --warmup 5 --steps 40 --no-cpu-baseline"
      [ $c = c2 ] && args="--warmup 5 --steps 50 --no-cpu-baseline"
      env $(echo $envs | tr ',' ' ') timeout 600 python bench.py $args | sed "s/^/$name $c /" >> gpurun_out/ablib.jsonl
    done
  done
done 2> gpurun_out/ablib.err
