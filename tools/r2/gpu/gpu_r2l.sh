#!/bin/bash
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_train_sparse.py tests/test_gpu_exchange.py tests/test_gpu_gcn.py > gpurun_out/r2l_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2l_pytest.txt
run() { name=$1; shift; timeout 900 python bench.py --no-cpu --no-e2e --no-ablation "$@" > gpurun_out/r2l_$name.json 2> gpurun_out/r2l_$name.err; }
run papersq --config papers-q --steps 5
PGCN_SPMM_TABLE="12=16,1,8,3" run papersq_16183 --config papers-q --steps 5
run reddit
run products --config products
run yelp --config yelp --smooth gf
tail -2 gpurun_out/r2l_pytest.txt
