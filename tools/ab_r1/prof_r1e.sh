# r1e: profiles of the current build (Reddit-shaped step after 3 warm-up steps): launch list with
# DRAM bytes, then ncu --set full of the wide and narrow SpMMs (fwd + transposed), the layer-1 dW
# GEMM, a layer-2 fwd GEMM and a dropout launch.
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
F="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv $B > gpurun_out/launch_bench_r1e.json 2>&1
timeout 600 $F -k regex:k_spmm_fwd -s 24 -c 1 -o gpurun_out/r1e_spmm_fwd_wide $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_fwd -s 30 -c 1 -o gpurun_out/r1e_spmm_fwd_narrow $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_bwd -s 24 -c 1 -o gpurun_out/r1e_spmm_bwd_narrow $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_bwd -s 26 -c 1 -o gpurun_out/r1e_spmm_bwd_wide $B > /dev/null 2>&1
timeout 600 $F -k regex:k_umma_gemm -s 103 -c 1 -o gpurun_out/r1e_gemm_dw1 $B > /dev/null 2>&1
timeout 600 $F -k regex:k_umma_gemm -s 82 -c 1 -o gpurun_out/r1e_gemm_fwd2 $B > /dev/null 2>&1
timeout 600 $F -k regex:k_dropout -s 12 -c 1 -o gpurun_out/r1e_dropout $B > /dev/null 2>&1
timeout 400 python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err
ls -la gpurun_out | tail -10
