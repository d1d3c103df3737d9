# r1d: ncu --set full of the current build (Reddit-shaped step after 3 warm-up steps): wide and
# narrow SpMM (fwd + transposed), the layer-1 dW GEMM; then every BASELINE config on one GPU.
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
F="ncu --set full --clock-control none --import-source on"
timeout 600 $F -k regex:k_spmm_fwd -s 24 -c 1 -o gpurun_out/r1d_spmm_fwd_wide $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_fwd -s 30 -c 1 -o gpurun_out/r1d_spmm_fwd_narrow $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_bwd -s 24 -c 1 -o gpurun_out/r1d_spmm_bwd_narrow $B > /dev/null 2>&1
timeout 600 $F -k regex:k_spmm_bwd -s 26 -c 1 -o gpurun_out/r1d_spmm_bwd_wide $B > /dev/null 2>&1
timeout 600 $F -k regex:k_umma_gemm -s 103 -c 1 -o gpurun_out/r1d_gemm_dw1 $B > /dev/null 2>&1
timeout 600 $F -k regex:k_dropout -s 12 -c 1 -o gpurun_out/r1d_dropout $B > /dev/null 2>&1
bash tools/all_configs.sh > gpurun_out/r1d_all_configs.txt 2>&1
ls -la gpurun_out | tail -9
