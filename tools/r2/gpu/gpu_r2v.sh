#!/bin/bash
# regression after the multi-process PUSH change: exchange / lean suites, smoke, push bench on one GPU
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2v; mkdir -p $O
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_exchange.py tests/test_gpu_lean.py tests/test_gpu_multigpu.py > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py --transport push --no-cpu --no-e2e > $O/reddit_push.json 2> $O/reddit_push.err
timeout 300 python bench.py --gpus 2 > $O/gpus2.json 2> $O/gpus2.err; echo "gpus2 rc=$?" >> $O/gpus2.err
tail -2 $O/pytest.txt; tail -1 $O/smoke.txt; tail -2 $O/gpus2.err; head -c 300 $O/gpus2.json
