# r1n: dropout with two loads in flight per thread
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1n.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1n.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1n.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r1n.txt
for C in "reddit" "products" "yelp --smooth gf" "reddit --model gcn"; do
  timeout 400 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('%-24s %8.2f ep/s %8.2f ms dropout %.3f ms (%.0f GB/s)' % ('$C', d['value'], d['ms_per_step'], d['breakdown']['dropout']['ms_per_step'], d['breakdown']['dropout']['GBps']))"
done
