# Every BASELINE config that fits one GPU, 2 partitions on 1 GPU (local transport); fp32 tier, then
# the bf16 gather tier (--gather bf16) of the same configs.
for C in "cora" "reddit" "reddit --no-tiles" "products" "papers-q" "yelp --smooth gf" "reddit --mode vanilla" "reddit --smooth gf" "reddit --model gcn" \
         "reddit --gather bf16" "products --gather bf16" "yelp --smooth gf --gather bf16" "reddit --gather bf16 --gemm bf16"; do
  timeout 400 python bench.py --config $C --steps 10 --warmup 3 --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); r=d['roofline']; c=d.get('cpu_baseline') or {}
print('%-36s %8.2f ep/s %8.2f ms  top=%s %.0f GB/s frac=%.2f  oracle %.4g ep/s (%s cores)' % ('$C', d['value'], d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], c.get('value', float('nan')), c.get('cores')))
print('   ', json.dumps({k: round(v['ms_per_step'], 2) for k, v in d['breakdown'].items()}))"
done
