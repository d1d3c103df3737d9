timeout 900 python -m pytest tests/test_gpu_train_sparse.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_cl.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_cl.txt | grep -v "^$" | tail -8
timeout 900 python bench.py --config papers-q --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_papers_cl.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_papers_cl.json')); print('papers-q', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items()})" || tail -5 gpurun_out/bench_papers_cl.json
timeout 300 python bench.py --config products --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_products_cl.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_products_cl.json')); print('products', round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['breakdown'].items()})" || tail -5 gpurun_out/bench_products_cl.json
