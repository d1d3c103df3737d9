timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles6.txt 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_tiles6.txt
run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/b6.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/b6.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -5 gpurun_out/b6.json
}
for rep in 1 2; do
run "PGCN_TILE_CONCURRENT=1"
run "PGCN_TILE_CONCURRENT=0"
run "PGCN_TILE_CONCURRENT=1" "--gather bf16"
run "PGCN_TILE_CONCURRENT=0" "--gather bf16"
done
run "PGCN_TILE_CONCURRENT=1 PGCN_TC_SPMM_ORDER=0"
run "PGCN_TILE_CONCURRENT=1 PGCN_TC_SPMM_TS=0"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_tiles6.csv $B > /dev/null 2>&1
