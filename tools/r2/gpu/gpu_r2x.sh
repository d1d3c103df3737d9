#!/bin/bash
# dW with two CTAs per SM (PGCN_TC_DW_CTAS=2, split plan sized for 2 x SMs): correctness + A/B
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2x; mkdir -p $O
PGCN_TC_DW_CTAS=2 timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_parity.py > $O/pytest_ctas2.txt 2>&1; echo "rc=$?" >> $O/pytest_ctas2.txt
tail -2 $O/pytest_ctas2.txt
if grep -q "rc=0" $O/pytest_ctas2.txt; then
  for c in 2 1; do
    for cfg in papers-q products reddit yelp; do
      sm=""; [ $cfg = yelp ] && sm="--smooth gf"
      PGCN_TC_DW_CTAS=$c timeout 900 python bench.py --config $cfg $sm --no-cpu --no-e2e --no-ablation --steps 10 > $O/${cfg}_c$c.json 2> $O/${cfg}_c$c.err
    done
  done
fi
ls $O
