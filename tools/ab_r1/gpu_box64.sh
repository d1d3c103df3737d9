PGCN_TC_SPMM_BOX64=1 timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_box64.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_box64.txt
run() {
  env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/bx.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/bx.json')); print('$1 $2', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items() if v['ms_per_step'] > 0.5})" || tail -3 gpurun_out/bx.json
}
run "PGCN_TC_SPMM_BOX64=0"
run "PGCN_TC_SPMM_BOX64=1"
run "PGCN_TC_SPMM_BOX64=0" "--gather bf16"
run "PGCN_TC_SPMM_BOX64=1" "--gather bf16"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_box.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 24 -c 1 -o gpurun_out/box_tc $B > /dev/null 2>&1
