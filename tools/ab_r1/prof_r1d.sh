# Re-validation after container restore: GPU tests, smoke, bench, launch list of one timed step.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r1d.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/gpu_tests_r1d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; cat gpurun_out/bench_r1d.json
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv $B > gpurun_out/launch_bench_r1d.json 2>&1
ls -la gpurun_out | tail -8
