set -x
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles3.txt 2>&1; echo "rc=$?"
tail -25 gpurun_out/pytest_tiles3.txt
for bn in 128 256; do
PGCN_TC_SPMM_BN=$bn timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_tiles3_$bn.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_tiles3_$bn.json')); print('BN $bn', d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items()})"
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --gather bf16 > gpurun_out/bench_tiles3_bf16.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_tiles3_bf16.json')); print('bf16', d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items()})"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_tiles3.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 12 -c 1 -o gpurun_out/tiles3_tc $B > /dev/null 2>&1
ls gpurun_out
