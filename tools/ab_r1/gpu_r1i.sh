# r1i: final round-1 measurement of the defaults: GPU suite, smoke, bench, launch list, ncu captures, all configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1i.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_r1i.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1i.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r1i.txt
timeout 400 python bench.py > gpurun_out/bench_r1i.json 2> gpurun_out/bench_r1i.err; echo "bench rc=$?"
head -c 2500 gpurun_out/bench_r1i.json; echo
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1i.json 2>&1; echo "ref rc=$?"; head -c 600 gpurun_out/bench_ref_r1i.json; echo
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
F="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1i.csv $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_tc -s 24 -c 1 -o gpurun_out/r1i_spmm_tc $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_fwd -s 20 -c 1 -o gpurun_out/r1i_spmm_fwd_light $B > /dev/null 2>&1
timeout 600 $F -k regex:k_umma_gemm -s 103 -c 1 -o gpurun_out/r1i_gemm $B > /dev/null 2>&1
timeout 600 $F -k regex:k_dropout -s 12 -c 1 -o gpurun_out/r1i_dropout $B > /dev/null 2>&1
bash tools/all_configs.sh > gpurun_out/all_configs_r1i.txt 2>&1
cat gpurun_out/all_configs_r1i.txt
