#!/bin/bash
# box CPU budget around a C5 run: cgroup quota / throttling counters, cores
mkdir -p gpurun_out
{
nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/cpu.stat 2>/dev/null
cat /sys/fs/cgroup/cpu/cpu.cfs_quota_us /sys/fs/cgroup/cpu/cpu.cfs_period_us /sys/fs/cgroup/cpu/cpu.stat 2>/dev/null
python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"
uptime
for i in 1 2 3; do timeout 600 python bench.py --workload c5 --warmup 5 --steps 40 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['worst_step']['ms'])"; cat /sys/fs/cgroup/cpu.stat 2>/dev/null | head -6; done
uptime
top -b -n 1 | head -25
} > gpurun_out/cg.txt 2>&1
