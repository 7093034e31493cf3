for b in 4096 65536; do for v in "" "--no-pipeline"; do for r in 1 2; do
 echo "== batch $b $v run $r"; timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 3 --cold --batch $b $v > gpurun_out/cold_$b$v.log 2>&1; echo rc=$?; tail -1 gpurun_out/cold_$b$v.log | cut -c1-200
done; done; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --cold --batch 4096 --no-pipeline 2>&1 | tail -2
