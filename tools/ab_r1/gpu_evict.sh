timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_evict.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_evict.txt
run() {
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $1 > gpurun_out/be.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/be.json')); print('$1', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 2.0})"
}
run ""
run ""
run "--gather bf16"
run "--config products"
run "--no-tiles"
run "--config papers-q --steps 4"
