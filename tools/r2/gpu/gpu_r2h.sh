#!/bin/bash
# round 2: column-chunked (L2-resident) gathers -- parity with chunking forced on small graphs, Reddit sweep
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
PGCN_SPMM_L2MB=1 timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_train_sparse.py tests/test_gpu_gcn.py tests/test_gpu_bf16_gather.py > gpurun_out/r2h_pytest_chunked.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2h_pytest_chunked.txt
for mb in 0 96 64 32 16; do
  PGCN_SPMM_L2MB=$mb timeout 600 python bench.py --no-cpu --no-e2e --no-ablation > gpurun_out/r2h_reddit_l2mb$mb.json 2> gpurun_out/r2h_reddit_l2mb$mb.err
done
for mb in 0 64 32; do
  PGCN_SPMM_L2MB=$mb timeout 900 python bench.py --config products --no-cpu --no-e2e --no-ablation > gpurun_out/r2h_products_l2mb$mb.json 2> gpurun_out/r2h_products_l2mb$mb.err
done
tail -2 gpurun_out/r2h_pytest_chunked.txt
