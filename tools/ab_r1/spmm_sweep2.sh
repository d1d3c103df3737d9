for T in "" "151=32,5,1,2;64=32,2,4,4" "151=32,5,1,1;64=32,2,4,3" "151=32,6,1,3;64=32,2,2,4" "151=32,4,2,2;64=32,1,8,4" "151=32,5,1,3;64=32,2,4,2" "151=32,1,8,4;64=32,1,8,3"; do
  PGCN_SPMM_TABLE="$T" timeout 200 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T' or 'default', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
