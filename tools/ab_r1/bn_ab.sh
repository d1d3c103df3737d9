# FWD/DA n-tile cap A/B (PGCN_TC_BNMAX) on the Reddit- and Yelp-shaped steps.
for C in "reddit" "yelp --smooth gf"; do
  for BN in 256 128 64; do
    PGCN_TC_BNMAX=$BN timeout 300 python bench.py --config $C --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-18s BN<=%-4s %7.2f ms/step ' % ('$C', '$BN', d['ms_per_step']) + ' '.join('%s %.2f' % (k, v['ms_per_step']) for k, v in b.items() if k.startswith('gemm')))"
  done
done
