run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/bt.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bt.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -3 gpurun_out/bt.json
}
run "PGCN_TF_OFF=0"
run "PGCN_TF_OFF=2"
run "PGCN_TF_OFF=16"
run "PGCN_TF_OFF=0" "--gather bf16"
run "PGCN_TF_OFF=2" "--gather bf16"
run "PGCN_TF_OFF=0" "--model gcn"
run "PGCN_TF_OFF=2" "--model gcn"
