#!/bin/bash
# loss over the train row list (few train rows): parity suites + products / Yelp / Reddit bench
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2w; mkdir -p $O
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_train_sparse.py tests/test_gpu_parity.py tests/test_gpu_fullsize_step.py tests/test_gpu_exchange.py tests/test_gpu_lean.py tests/test_gpu_gcn.py > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for cfg in products reddit; do
  timeout 900 python bench.py --config $cfg --no-cpu --no-e2e --no-ablation > $O/$cfg.json 2> $O/$cfg.err
done
tail -2 $O/pytest.txt
