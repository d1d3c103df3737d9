# r1q: final round-1 measurement of HEAD (branch-free dropout mask in k_dropout and the transposed-SpMM epilogues)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1q.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1q.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1q.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r1q.txt
timeout 400 python bench.py > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err; echo "bench rc=$?"
head -c 1500 gpurun_out/bench_r1q.json; echo
timeout 400 python bench.py --impl reference > gpurun_out/bench_reference_r1q.json 2> gpurun_out/bench_reference_r1q.err; echo "ref rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1q.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 24 -c 1 -o gpurun_out/r1q_spmm_tc $B > /dev/null 2>&1
ncu -i gpurun_out/r1q_spmm_tc.ncu-rep --page raw --csv > gpurun_out/r1q_spmm_tc_raw.csv 2>/dev/null
P="python bench.py --config papers-q --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1q_papers.csv $P > /dev/null 2>&1
bash tools/all_configs.sh > gpurun_out/all_configs_r1q.txt 2>&1
cat gpurun_out/all_configs_r1q.txt
