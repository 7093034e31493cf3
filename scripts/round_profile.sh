#!/bin/bash
# Run on the GPU box (via gpurun): everything a round's profiles/ needs —
# headline bench line + launch list + ncu --set full capture (gpu_profile.sh),
# the C1/C3/C4/C5 config lines, and the Table-1 / §8(a) operator tables.
TAG=${1:-r09}
mkdir -p gpurun_out
bash scripts/gpu_profile.sh "$TAG"
: > gpurun_out/configs_${TAG}.jsonl
for w in c1 c3 c4 c5; do
  timeout 600 python bench.py --workload $w --warmup 5 $([ $w = c1 ] || echo --steps 20) >> gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/cfg_${w}.err
done
timeout 300 python ops_bench.py > gpurun_out/ops_${TAG}.txt 2>&1
timeout 300 python ops_bench.py --rows > gpurun_out/ops_rows_${TAG}.txt 2>&1
ls -la gpurun_out
