run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bsh.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bsh.json')); print('$1', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 5.0})"
}
for i in 1 2 3; do
run "X=0"
run "PGCN_SPMM_TABLE=64=32,2,4,3"
run "PGCN_SPMM_TABLE=64=32,2,4,4"
done
