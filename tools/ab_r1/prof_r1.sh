set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_fwd -s 24 -c 4 -o gpurun_out/prof_spmm_fwd $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bwd -s 18 -c 2 -o gpurun_out/prof_spmm_bwd $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 60 -c 4 -o gpurun_out/prof_gemm $B > /dev/null 2>&1
ls -la gpurun_out
