# bf16 gather tier: FHADD vs FADD2-unpack A/B and shape sweep (Reddit-shaped step, --gather bf16).
bash tools/ab_run.sh "--gather bf16" tools/ab/libpgcn_fadd2.so -
for T in "1000032=32,1,8,4" "1000032=32,1,12,3" "1000006=8,1,16,2" "1000006=16,1,8,4" "1000006=16,1,16,2"; do
  PGCN_SPMM_TABLE="$T" timeout 200 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e --gather bf16 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --gather bf16"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1f16.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fwd16 -s 24 -c 1 -o gpurun_out/r1f_spmm16_fwd_wide $B > /dev/null 2>&1
