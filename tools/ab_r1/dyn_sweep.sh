for D in 0 1; do
  PGCN_SPMM_DYN=$D timeout 200 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('dyn=$D %7.2f ms/step  fwd %6.2f  bwd %6.2f' % (d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
done
