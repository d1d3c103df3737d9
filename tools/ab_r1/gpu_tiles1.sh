# first run of the tensor-core tile aggregation: unit parity, then bench with/without tiles
set -x
timeout 600 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles1.txt 2>&1; echo "rc=$?"
tail -30 gpurun_out/pytest_tiles1.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_tiles1.json 2> gpurun_out/bench_tiles1.err; echo "rc=$?"
cat gpurun_out/bench_tiles1.json; tail -5 gpurun_out/bench_tiles1.err
