#!/bin/bash
# 16-row k-blocks for the 3xTF32 dW GEMM (PGCN_TC_DW16): tests + A/B
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2t; mkdir -p $O
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py > $O/pytest_gemm.txt 2>&1; echo "rc=$?" >> $O/pytest_gemm.txt
tail -2 $O/pytest_gemm.txt
if grep -q "rc=0" $O/pytest_gemm.txt; then
  timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize_step.py tests/test_gpu_lean.py tests/test_gpu_gcn.py tests/test_gpu_train_sparse.py > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
  for dw in 1 0; do
    for cfg in reddit yelp products papers-q; do
      sm=""; [ $cfg = yelp ] && sm="--smooth gf"
      PGCN_TC_DW16=$dw timeout 900 python bench.py --config $cfg $sm --no-cpu --no-e2e --no-ablation --steps 10 > $O/${cfg}_dw$dw.json 2> $O/${cfg}_dw$dw.err
    done
  done
fi
tail -2 $O/pytest.txt
