#!/bin/bash
# round 2: papers-e SpMM shape sweep (ld4 = 12), steady-state ncu capture of the papers aggregation, all configs
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
for sh in default 4,3,4,3 4,3,8,2 4,3,2,4 8,2,4,3 8,2,8,2; do
  if [ $sh = default ]; then unset PGCN_SPMM_TABLE; else export PGCN_SPMM_TABLE="12=$sh"; fi
  timeout 900 python bench.py --config papers-e --no-cpu --no-e2e --no-ablation --steps 5 > gpurun_out/r2f_papers_e_$sh.json 2> gpurun_out/r2f_papers_e_$sh.err
done
unset PGCN_SPMM_TABLE
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_bwd" --launch-skip 14 --launch-count 4 -o gpurun_out/r2f_papers_e_spmm python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2f_ncu_spmm.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_umma_gemm" --launch-skip 30 --launch-count 12 -o gpurun_out/r2f_papers_e_gemm python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2f_ncu_gemm.log 2>&1
bash tools/r2/all_configs.sh
