# r1r: k_grad_reduce walks (row, float4) with RowCursor instead of a 64-bit divide per item
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1r.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1r.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1r.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r1r.txt
for C in "reddit" "products" "yelp --smooth gf" "papers-q"; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-24s %8.2f ep/s %8.2f ms grad_reduce %.3f ms (%.0f GB/s)' % ('$C', d['value'], d['ms_per_step'], b['grad_reduce']['ms_per_step'], b['grad_reduce']['GBps']))"
done
