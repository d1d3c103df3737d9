timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_train_sparse.py tests/test_gpu_gcn.py -x -q > gpurun_out/pytest_colsum.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_colsum.txt
run() {
  timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bc.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bc.json')); print('$1', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -3 gpurun_out/bc.json
}
run reddit
run reddit
run products
run yelp
run papers-q
