# tile aggregation: parity tests, launch list, one full ncu capture of a wide k_spmm_tc launch
set -x
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles2.txt 2>&1; echo "rc=$?"
tail -5 gpurun_out/pytest_tiles2.txt
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_tiles2.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 12 -c 1 -o gpurun_out/tiles2_tc $B > /dev/null 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --gather bf16 > gpurun_out/bench_tiles2_bf16.json 2>&1
cat gpurun_out/bench_tiles2_bf16.json | head -c 600
