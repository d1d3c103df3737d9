timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_train_sparse.py -x -q > gpurun_out/pytest_gemm2.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gemm2.txt
run() {
  env $1 timeout 600 python bench.py --config $2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bg.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bg.json')); print('$1 $2', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -3 gpurun_out/bg.json
}
run "PGCN_TC_GEMM_CTAS=1" products
run "PGCN_TC_GEMM_CTAS=2" products
run "PGCN_TC_GEMM_CTAS=1" yelp
run "PGCN_TC_GEMM_CTAS=2" yelp
run "PGCN_TC_GEMM_CTAS=1" papers-q
run "PGCN_TC_GEMM_CTAS=2" papers-q
run "PGCN_TC_GEMM_CTAS=2" reddit
