# Round-1 profile of the current kernels (run under gpurun).  Launch list of one timed step after 3
# warm-up steps, then ncu --set full of the SpMMs and the tcgen05 GEMM of that step.
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $B > gpurun_out/launch_bench_r1b.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fwd -s 24 -c 8 -o gpurun_out/prof_spmm_fwd_r1b $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_bwd -s 18 -c 2 -o gpurun_out/prof_spmm_bwd_r1b $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 66 -c 6 -o gpurun_out/prof_umma_r1b $B > /dev/null 2>&1
timeout 400 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err
ls -la gpurun_out | tail -8
