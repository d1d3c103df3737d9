# r1g (session 3 re-entry): gpu tests, default bench, launch list of the current build.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1g.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1g.txt
timeout 400 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err; echo "bench rc=$?"
cat gpurun_out/bench_r1g.json
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1g.csv $B > gpurun_out/launch_bench_r1g.json 2>&1
bash tools/all_configs.sh > gpurun_out/all_configs_r1g.txt 2>&1
cat gpurun_out/all_configs_r1g.txt
