mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --workload c3 --steps 3 --warmup 2 --c3-rows 2e7 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python -c "
import cProfile, pstats, sys
sys.argv=['bench.py','--workload','c5','--steps','3','--warmup','2','--no-cpu-baseline']
import bench
cProfile.run('bench.main()', '/tmp/c5.prof')
p=pstats.Stats('/tmp/c5.prof'); p.sort_stats('cumtime').print_stats(45)
" > gpurun_out/c5_cprofile.txt 2>&1
ls -la gpurun_out | tail -5
