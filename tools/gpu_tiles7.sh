run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/b7.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/b7.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -5 gpurun_out/b7.json
}
run "PGCN_TILE_CONCURRENT=0"
run "PGCN_TILE_CONCURRENT=1"
run "PGCN_TILE_CONCURRENT=1 PGCN_SIDE_BLOCKS=296"
run "PGCN_TILE_CONCURRENT=1 PGCN_SIDE_BLOCKS=74"
run "PGCN_TILE_CONCURRENT=0" "--gather bf16"
run "PGCN_TILE_CONCURRENT=1" "--gather bf16"
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q -k "light_mix" > gpurun_out/pytest_tiles7.txt 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_tiles7.txt
