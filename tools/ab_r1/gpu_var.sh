timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_var.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_var.txt
for i in 1 2; do
timeout 400 python bench.py --no-cpu > gpurun_out/bv.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bv.json')); print('default', round(d['value'],2), round(d['ms_per_step'],2), d['clocks'], {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})"
timeout 400 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/bv.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bv.json')); print('short', round(d['value'],2), round(d['ms_per_step'],2), d['clocks'], {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})"
timeout 400 python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/bv.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bv.json')); print('20/5 noe2e', round(d['value'],2), round(d['ms_per_step'],2), d['clocks'], {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})"
done
