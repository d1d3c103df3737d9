# Per-launch view of the 26 tcgen05 GEMM launches of one Reddit step (after 3 warm-up steps) and a
# full-set capture of the layer-1 and layer-2 dW launches (run under gpurun).
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu $*"
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:k_umma_gemm -s 78 -c 26 --log-file gpurun_out/gemm_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 90 -c 1 -o gpurun_out/prof_dw4 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 102 -c 1 -o gpurun_out/prof_dw1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 94 -c 1 -o gpurun_out/prof_dw3 $B > /dev/null 2>&1
ls -la gpurun_out | tail -5
