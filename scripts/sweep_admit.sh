for e in 0 1; do for v in "" "--prefetch-early"; do
 echo "== coop=$e $v"; SKB_ADMIT_COOP=$e timeout 300 python bench.py --no-cpu-baseline --steps 50 $v > gpurun_out/sw_$e$v.log 2>&1; tail -1 gpurun_out/sw_$e$v.log | cut -c1-200
 python - "gpurun_out/sw_$e$v.log" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["e2e"]["value"]/1e9,3), {k:round(x,3) for k,x in d["kernels_ms"].items()})
except Exception as ex: print("ERR", ex)
PY
done
echo "== cold coop=$e"; SKB_ADMIT_COOP=$e timeout 300 python bench.py --no-cpu-baseline --steps 20 --cold > gpurun_out/swc_$e.log 2>&1; tail -2 gpurun_out/swc_$e.log | cut -c1-600
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
