for C in "reddit" "products" "yelp --smooth gf"; do
  timeout 400 python bench.py --config $C --gemm bf16 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('bf16 %-18s %8.2f ep/s %8.2f ms' % ('$C', d['value'], d['ms_per_step']), json.dumps({k: round(v['ms_per_step'], 2) for k, v in d['breakdown'].items()}))"
done
