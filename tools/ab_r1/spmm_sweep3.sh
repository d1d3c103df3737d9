# In-situ sweep of narrow-width SpMM shapes (ld4 11 = Reddit classes 41) and the 256-wide
# occupancy, after the neighbour-id prefetch change.  Full Reddit-shaped bench step per table.
for T in "" "11=16,1,16,2" "11=16,1,12,3" "11=32,1,16,2" "11=32,1,12,3" "11=16,1,16,3" "64=32,2,4,3" "64=32,1,8,3" "64=32,1,16,2"; do
  PGCN_SPMM_TABLE="$T" timeout 200 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-40s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$T' or 'default', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
