timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_final.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.txt
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final.json 2>&1; echo "ref rc=$?"; head -c 300 gpurun_out/bench_ref_final.json
