set -x
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles4.txt 2>&1; echo "rc=$?"
tail -4 gpurun_out/pytest_tiles4.txt
for cfg in "PGCN_TC_SPMM_TS=1" "PGCN_TC_SPMM_TS=0" "PGCN_TC_SPMM_TS=1 PGCN_TC_SPMM_BN=64" "PGCN_TC_SPMM_TS=1 PGCN_TC_SPMM_BN=192"; do
env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b4.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/b4.json')); print('$cfg', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items()})" || tail -5 gpurun_out/b4.json
done
for cfg in "PGCN_TC_SPMM_TS=1" "PGCN_TC_SPMM_TS=1 PGCN_TC_SPMM_BN=128"; do
env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --gather bf16 > gpurun_out/b4.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/b4.json')); print('bf16 $cfg', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items()})" || tail -5 gpurun_out/b4.json
done
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_tiles4.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 12 -c 1 -o gpurun_out/tiles4_tc $B > /dev/null 2>&1
