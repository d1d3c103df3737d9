run() {
  timeout 400 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 $1 > gpurun_out/bm.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bm.json')); print('$1', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 1.0})"
}
for tm in 96 48 160 256 400 600 96; do run "--tile-min $tm"; done
