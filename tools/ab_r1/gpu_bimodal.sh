for c in 2 2 2 2 2 2 1 1 1 1; do
PGCN_TC_SPMM_CTAS=$c timeout 400 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/bb.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bb.json')); print('ctas $c', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 1.0})"
done
for c in 1 2 3; do
timeout 400 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 --no-tiles > gpurun_out/bb.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bb.json')); print('no-tiles', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 1.0})"
done
