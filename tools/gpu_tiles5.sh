timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles5.txt 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_tiles5.txt
run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/b5.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/b5.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -5 gpurun_out/b5.json
}
run "PGCN_LIGHT_STRIPE_KB=0"
run "PGCN_LIGHT_STRIPE_KB=65536"
run "PGCN_LIGHT_STRIPE_KB=32768"
run "PGCN_LIGHT_STRIPE_KB=131072"
run "PGCN_LIGHT_STRIPE_KB=65536 PGCN_TC_SPMM_ORDER=0"
run "PGCN_LIGHT_STRIPE_KB=0 PGCN_TC_SPMM_ORDER=0"
run "PGCN_LIGHT_STRIPE_KB=65536" "--gather bf16"
run "PGCN_LIGHT_STRIPE_KB=32768" "--gather bf16"
run "PGCN_LIGHT_STRIPE_KB=0" "--gather bf16"
run "PGCN_LIGHT_STRIPE_KB=65536 PGCN_TC_SPMM_ORDER=0" "--gather bf16"
