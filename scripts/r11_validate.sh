#!/bin/bash
# HEAD validation on the GPU box: full GPU suite, smoke, headline bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
: > gpurun_out/cfg.jsonl
for w in c5 c4; do
  timeout 600 python bench.py --workload $w --warmup 5 --steps 20 --no-cpu-baseline 2>>gpurun_out/cfg.err >> gpurun_out/cfg.jsonl
done
tail -3 gpurun_out/gpu_tests.log
