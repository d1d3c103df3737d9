# Dynamic SpMM scheduler: edges per atomic grab (PGCN_SPMM_GRAB) on Reddit / products / papers-q.
for C in reddit products papers-q; do
  for G in 64 128 256 512; do
    PGCN_SPMM_GRAB=$G timeout 300 python bench.py --config $C --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-10s grab %-5s %7.2f ms/step  fwd %6.2f  bwd %6.2f' % ('$C', '$G', d['ms_per_step'], b['spmm_fwd']['ms_per_step'], b['spmm_bwd']['ms_per_step']))"
  done
done
