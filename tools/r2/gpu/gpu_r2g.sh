#!/bin/bash
# round 2: dW stage change validation + timing, papers-e SpMM shape sweep, steady-state ncu of the papers
# aggregation and GEMMs (exported to CSV on the box: full reports exceed the copy-back limit), all configs
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_gemm.py "tests/test_gpu_fullsize_step.py" > gpurun_out/r2g_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_pytest.txt
timeout 600 python tools/r2/dw_chain.py > gpurun_out/r2g_dw_chain.jsonl 2> gpurun_out/r2g_dw_chain.err
for sh in default 4,3,4,3 4,3,8,2 4,3,2,4 8,2,4,3 8,2,8,2; do
  if [ $sh = default ]; then unset PGCN_SPMM_TABLE; else export PGCN_SPMM_TABLE="12=$sh"; fi
  timeout 900 python bench.py --config papers-e --no-cpu --no-e2e --no-ablation --steps 5 > gpurun_out/r2g_papers_e_$sh.json 2> gpurun_out/r2g_papers_e_$sh.err
done
unset PGCN_SPMM_TABLE
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_bwd" --launch-skip 14 --launch-count 3 -o /tmp/r2g_spmm python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2g_ncu_spmm.log 2>&1
ncu -i /tmp/r2g_spmm.ncu-rep --page raw --csv > gpurun_out/r2g_papers_e_spmm_raw.csv 2>/dev/null
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_umma_gemm" --launch-skip 30 --launch-count 8 -o /tmp/r2g_gemm python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2g_ncu_gemm.log 2>&1
ncu -i /tmp/r2g_gemm.ncu-rep --page raw --csv > gpurun_out/r2g_papers_e_gemm_raw.csv 2>/dev/null
bash tools/r2/all_configs.sh
du -sh gpurun_out
