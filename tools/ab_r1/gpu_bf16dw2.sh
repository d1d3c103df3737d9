timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_bf16_gather.py -x -q > gpurun_out/pytest_bf16dw.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_bf16dw.txt
run() {
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $1 > gpurun_out/bb2.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bb2.json')); print('$1', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 1.0})"
}
run "--gather bf16 --gemm bf16"
run "--gather bf16"
run "--gather bf16 --gemm bf16"
run "--config yelp --smooth gf --gather bf16 --gemm bf16"
