# r1k: final round-1 measurement (defaults incl. the dW column-sum split)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1k.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1k.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1k.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r1k.txt
timeout 400 python bench.py > gpurun_out/bench_r1k.json 2> gpurun_out/bench_r1k.err; echo "bench rc=$?"
head -c 1500 gpurun_out/bench_r1k.json; echo
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1k.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 24 -c 1 -o gpurun_out/r1k_spmm_tc $B > /dev/null 2>&1
P="python bench.py --config papers-q --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1k_papers.csv $P > /dev/null 2>&1
bash tools/all_configs.sh > gpurun_out/all_configs_r1k.txt 2>&1
cat gpurun_out/all_configs_r1k.txt
