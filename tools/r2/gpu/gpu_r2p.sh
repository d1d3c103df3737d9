#!/bin/bash
# producer-written M_lo (3xTF32 pre-split operand): GPU tests, bench A/B (PGCN_PRESPLIT=0 vs 1) on Reddit / Yelp
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2p; mkdir -p $O
timeout 2400 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_lean.py tests/test_gpu_parity.py tests/test_gpu_gcn.py tests/test_gpu_train_sparse.py tests/test_gpu_exchange.py tests/test_gpu_gemm.py tests/test_gpu_fullsize_step.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for ps in 1 0; do
  PGCN_PRESPLIT=$ps timeout 900 python bench.py --no-cpu --no-e2e --no-ablation > $O/reddit_ps$ps.json 2> $O/reddit_ps$ps.err
  PGCN_PRESPLIT=$ps timeout 900 python bench.py --config yelp --smooth gf --no-cpu --no-e2e --no-ablation > $O/yelp_ps$ps.json 2> $O/yelp_ps$ps.err
done
PGCN_PRESPLIT=1 timeout 900 python bench.py --config products --no-cpu --no-e2e --no-ablation > $O/products_ps1.json 2> $O/products_ps1.err
tail -3 $O/pytest.txt
