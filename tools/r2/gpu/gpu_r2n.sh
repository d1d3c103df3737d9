#!/bin/bash
# re-entry check of HEAD: GPU tests, smoke, default bench twice
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2n; mkdir -p $O
nvidia-smi -L > $O/gpu.txt; nproc >> $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --config yelp --smooth gf --no-e2e --no-cpu > $O/yelp.json 2> $O/yelp.err
tail -3 $O/pytest_gpu.txt; tail -2 $O/smoke.txt; cat $O/bench.json | head -c 3000
