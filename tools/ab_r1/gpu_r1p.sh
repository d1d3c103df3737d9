# r1p: drop4 in the transposed-SpMM epilogues, scale only when dropout is on
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1p.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1p.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1p.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r1p.txt
for C in "reddit" "products" "yelp --smooth gf" "papers-q" "reddit --gather bf16" "products --gather bf16"; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-24s %8.2f ep/s %8.2f ms spmm_bwd %.3f ms dropout %.3f ms' % ('$C', d['value'], d['ms_per_step'], b['spmm_bwd']['ms_per_step'], b.get('dropout', {}).get('ms_per_step', 0)))"
done
