# r1h: full GPU suite, default bench, launch list + ncu full captures of the tile path, all configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1h.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1h.txt
timeout 400 python bench.py > gpurun_out/bench_r1h.json 2> gpurun_out/bench_r1h.err; echo "bench rc=$?"
head -c 3000 gpurun_out/bench_r1h.json; echo
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
F="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_tc -s 12 -c 1 -o gpurun_out/r1h_spmm_tc $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_fwd -s 20 -c 1 -o gpurun_out/r1h_spmm_fwd_light $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_bwd -s 24 -c 1 -o gpurun_out/r1h_spmm_bwd_light $B > /dev/null 2>&1
timeout 600 $F -k regex:k_split_bf16 -s 12 -c 1 -o gpurun_out/r1h_split $B > /dev/null 2>&1
bash tools/all_configs.sh > gpurun_out/all_configs_r1h.txt 2>&1
cat gpurun_out/all_configs_r1h.txt
