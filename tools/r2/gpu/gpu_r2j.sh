#!/bin/bash
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_train_sparse.py tests/test_gpu_tiles.py tests/test_gpu_parity.py > gpurun_out/r2j_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2j_pytest.txt
timeout 600 python bench.py --no-cpu > gpurun_out/r2j_reddit.json 2> gpurun_out/r2j_reddit.err
timeout 900 python bench.py --config papers-q --no-cpu --steps 5 > gpurun_out/r2j_papersq.json 2> gpurun_out/r2j_papersq.err
tail -2 gpurun_out/r2j_pytest.txt
