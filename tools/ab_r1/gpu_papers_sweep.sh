run() {
  env $1 timeout 600 python bench.py --config papers-q --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/bp.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bp.json')); print('$1', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 1})" || tail -3 gpurun_out/bp.json
}
run "X=1"
run "PGCN_SPMM_TABLE=12=4,3,4,4"
run "PGCN_SPMM_TABLE=12=4,3,8,3"
run "PGCN_SPMM_TABLE=12=8,2,4,4"
run "PGCN_SPMM_TABLE=12=8,1,8,4"
