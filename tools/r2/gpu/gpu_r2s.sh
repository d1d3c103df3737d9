#!/bin/bash
# 16-element k-blocks for every 3xTF32 K-major GEMM (PGCN_TC_BK16=2) vs only 256-wide n-tiles (1): tests + A/B
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2s; mkdir -p $O
PGCN_TC_BK16=2 timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_parity.py > $O/pytest_bk2.txt 2>&1; echo "rc=$?" >> $O/pytest_bk2.txt
tail -2 $O/pytest_bk2.txt
if grep -q "rc=0" $O/pytest_bk2.txt; then
  for bk in 2 1; do
    for cfg in products papers-q reddit; do
      PGCN_TC_BK16=$bk timeout 900 python bench.py --config $cfg --no-cpu --no-e2e --no-ablation --steps 10 > $O/${cfg}_bk$bk.json 2> $O/${cfg}_bk$bk.err
    done
  done
fi
ls $O
