#!/bin/bash
# 16-element k-blocks (SW64) for the 3xTF32 K-major GEMMs with 256-wide n-tiles: tests + bench A/B
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2r; mkdir -p $O
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py > $O/pytest_gemm.txt 2>&1; echo "rc=$?" >> $O/pytest_gemm.txt
tail -2 $O/pytest_gemm.txt
if grep -q "rc=0" $O/pytest_gemm.txt; then
  timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize_step.py tests/test_gpu_lean.py > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
  for bk in 1 0; do
    PGCN_TC_BK16=$bk timeout 900 python bench.py --no-cpu --no-e2e --no-ablation > $O/reddit_bk$bk.json 2> $O/reddit_bk$bk.err
    PGCN_TC_BK16=$bk timeout 900 python bench.py --config yelp --smooth gf --no-cpu --no-e2e --no-ablation > $O/yelp_bk$bk.json 2> $O/yelp_bk$bk.err
  done
  PGCN_TC_DW_BNMAX=128 timeout 900 python bench.py --no-cpu --no-e2e --no-ablation > $O/reddit_dwbn128.json 2> $O/reddit_dwbn128.err
  PGCN_TC_DW_BNMAX=128 timeout 900 python bench.py --config yelp --smooth gf --no-cpu --no-e2e --no-ablation > $O/yelp_dwbn128.json 2> $O/yelp_dwbn128.err
fi
tail -2 $O/pytest.txt
