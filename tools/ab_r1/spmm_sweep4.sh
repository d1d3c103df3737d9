# In-situ sweep after the 32-bit addressing / FADD2 rewrite (Reddit-shaped step).
for T in "" "64=32,2,8,2" "64=32,2,6,3" "64=32,2,4,3" "64=32,2,8,3" "11=16,1,16,2" "11=16,1,12,3" "11=16,1,16,3" "11=16,1,12,4"; do
  PGCN_SPMM_TABLE="$T" timeout 200 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T' or 'default', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
F="ncu --set full --clock-control none --import-source on"
timeout 600 $F -k regex:k_spmm_fwd -s 24 -c 1 -o gpurun_out/r1e_spmm_fwd_wide $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_fwd -s 30 -c 1 -o gpurun_out/r1e_spmm_fwd_narrow $B > /dev/null 2>&1
