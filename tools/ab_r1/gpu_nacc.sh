run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/bn.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bn.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 5.0})"
}
for i in 1 2; do
run "X=0"
run "PGCN_TC_SPMM_CTAS=1 PGCN_TC_SPMM_NACC1=1 PGCN_TC_SPMM_BN=256"
run "PGCN_TC_SPMM_CTAS=1 PGCN_TC_SPMM_NACC1=1 PGCN_TC_SPMM_BN=128"
done
PGCN_TC_SPMM_CTAS=1 PGCN_TC_SPMM_NACC1=1 PGCN_TC_SPMM_BN=256 timeout 600 python -m pytest tests/test_gpu_tiles.py -x -q -k "dense" > gpurun_out/pytest_nacc.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_nacc.txt
