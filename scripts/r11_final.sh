#!/bin/bash
# final HEAD check: full GPU suite, smoke, headline bench, Table-1 operators
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_final.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_final.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 300 python ops_bench.py > gpurun_out/ops_final.txt 2>&1
timeout 300 python ops_bench.py --rows > gpurun_out/ops_rows_final.txt 2>&1
tail -2 gpurun_out/gpu_tests_final.log; tail -1 gpurun_out/smoke_final.log
