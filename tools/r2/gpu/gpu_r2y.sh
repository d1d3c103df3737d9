#!/bin/bash
# dW two CTAs per SM where they fit (default now): suites + bench on every config shape
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2y; mkdir -p $O
timeout 1800 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_fullsize_step.py tests/test_gpu_lean.py tests/test_gpu_exchange.py tests/test_gpu_train_sparse.py tests/test_gpu_gcn.py > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -2 $O/pytest.txt
if grep -q "rc=0" $O/pytest.txt; then
  for cfg in papers-q products reddit yelp; do
    sm=""; [ $cfg = yelp ] && sm="--smooth gf"
    timeout 900 python bench.py --config $cfg $sm --no-cpu --no-e2e --no-ablation --steps 10 > $O/${cfg}.json 2> $O/${cfg}.err
  done
fi
ls $O
