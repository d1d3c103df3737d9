run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/bs.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bs.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 1.0})" || tail -3 gpurun_out/bs.json
}
run "X=1"
run "PGCN_SPMM_TABLE=64=32,2,4,4"
run "PGCN_SPMM_TABLE=64=32,2,4,3"
run "PGCN_SPMM_GRAB=64"
run "PGCN_SPMM_GRAB=256"
run "PGCN_SPMM_GRAB=512"
run "PGCN_SPMM_GRAB=1024"
run "X=1"
