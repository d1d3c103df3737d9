#!/bin/bash
# round 2: narrow-row gather kernels -- GPU parity suite, papers-q / Reddit / products with U = 8, 4, off
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest -q -x -p no:cacheprovider tests -m gpu --deselect tests/test_gpu_fullsize_step.py > gpurun_out/r2k_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k_pytest.txt
for me in 8 4 0; do
  PGCN_SPMM_ME=$me timeout 900 python bench.py --config papers-q --no-cpu --no-e2e --no-ablation --steps 5 > gpurun_out/r2k_papersq_me$me.json 2> gpurun_out/r2k_papersq_me$me.err
  PGCN_SPMM_ME=$me timeout 600 python bench.py --no-cpu --no-e2e --no-ablation > gpurun_out/r2k_reddit_me$me.json 2> gpurun_out/r2k_reddit_me$me.err
done
PGCN_SPMM_ME=8 timeout 600 python bench.py --config products --no-cpu --no-e2e --no-ablation > gpurun_out/r2k_products_me8.json 2> gpurun_out/r2k_products_me8.err
tail -2 gpurun_out/r2k_pytest.txt
