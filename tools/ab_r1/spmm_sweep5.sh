# In-situ sweep (Reddit 256-wide, products 100/128/48-wide, Yelp 300/512/100-wide) after the rewrite.
for T in "" "64=32,2,8,2" "64=32,2,12,2" "64=32,2,16,1" "64=32,2,10,2"; do
  PGCN_SPMM_TABLE="$T" timeout 200 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('reddit %-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T' or 'default', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
for T in "" "25=32,1,16,2;32=32,1,16,2" "12=16,1,16,2;25=32,1,16,2;32=32,1,16,2"; do
  PGCN_SPMM_TABLE="$T" timeout 300 python bench.py --config products --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('products %-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T' or 'default', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
for T in "" "75=32,3,4,2;128=32,4,4,2" "75=32,3,6,2;128=32,4,4,2;25=32,1,16,2"; do
  PGCN_SPMM_TABLE="$T" timeout 300 python bench.py --config yelp --smooth gf --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('yelp %-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T' or 'default', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
