#!/bin/bash
# lean-memory mode (N1(iii)): GPU tests, papers-q lean vs default, Reddit lean
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2o; mkdir -p $O
free -g > $O/host.txt; nproc >> $O/host.txt
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_lean.py tests/test_gpu_multigpu.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 900 python bench.py --config papers-q --lean --no-cpu --no-e2e --steps 10 > $O/papersq_lean.json 2> $O/papersq_lean.err
timeout 900 python bench.py --config papers-q --no-cpu --no-e2e --no-ablation --steps 10 > $O/papersq.json 2> $O/papersq.err
timeout 900 python bench.py --lean --no-cpu --no-e2e --no-ablation > $O/reddit_lean.json 2> $O/reddit_lean.err
tail -3 $O/pytest.txt
