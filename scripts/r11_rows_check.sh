#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "checked or deferred or distinct or scatter or adam or dropin or restore" > gpurun_out/rows_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rows_tests.log
tail -2 gpurun_out/rows_tests.log
timeout 300 python ops_bench.py 2>&1 | grep -E "gather|scatter|partition" | tail -8
