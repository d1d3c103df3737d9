#!/bin/bash
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_train_sparse.py > gpurun_out/r2m_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m_pytest.txt
timeout 600 python tools/r2/dw_chain.py > gpurun_out/r2m_dw_chain.jsonl 2> gpurun_out/r2m_dw_chain.err
timeout 900 python bench.py --config papers-q --no-cpu --no-e2e --no-ablation --steps 5 > gpurun_out/r2m_papersq.json 2> gpurun_out/r2m_papersq.err
PGCN_DW_MERGE=0 timeout 900 python bench.py --config papers-q --no-cpu --no-e2e --no-ablation --steps 5 > gpurun_out/r2m_papersq_nomerge.json 2> gpurun_out/r2m_papersq_nomerge.err
tail -2 gpurun_out/r2m_pytest.txt
