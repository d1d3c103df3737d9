run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/bc.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bc.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -3 gpurun_out/bc.json
}
run "PGCN_TC_SPMM_CTAS=2"
run "PGCN_TC_SPMM_CTAS=2 PGCN_TC_SPMM_BN=192"
run "PGCN_TC_SPMM_CTAS=1" "--gather bf16"
run "PGCN_TC_SPMM_CTAS=2" "--gather bf16"
run "PGCN_TC_SPMM_CTAS=2 PGCN_TC_SPMM_TS=0" "--gather bf16"
run "PGCN_TC_SPMM_CTAS=2 PGCN_TC_SPMM_BN=192" "--gather bf16"
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_ctas2.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ctas2.txt
PGCN_TC_SPMM_CTAS=1 timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q -k "vs_oracle and dense" > gpurun_out/pytest_ctas2b.txt 2>&1; echo "pytest1 rc=$?"; tail -2 gpurun_out/pytest_ctas2b.txt
