# Full-set captures of one Reddit step's J^(3) GEMM (layer-4 transform-first input gradient), the
# layer-2 dropout, and the layer-1 T GEMM (run under gpurun).
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu $*"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 91 -c 1 -o gpurun_out/prof_j4 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 78 -c 1 -o gpurun_out/prof_t1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dropout -s 26 -c 1 -o gpurun_out/prof_drop $B > /dev/null 2>&1
ls -la gpurun_out | tail -4
