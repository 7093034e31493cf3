#!/bin/bash
# Final profile set of round 2 (last session): GPU suite, then everything profiles/ needs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r11.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_r11.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r11.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r11.log
bash scripts/round_profile_r10.sh r11
