run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/bp.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bp.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -3 gpurun_out/bp.json
}
for dbg in 0 1 2 3; do run "PGCN_TC_SPMM_DBG=$dbg"; done
for dbg in 0 1 2 3; do run "PGCN_TC_SPMM_DBG=$dbg PGCN_TC_SPMM_BN=256"; done
for dbg in 0 1 2; do run "PGCN_TC_SPMM_DBG=$dbg" "--gather bf16"; done
