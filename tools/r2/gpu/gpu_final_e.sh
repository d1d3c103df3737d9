#!/bin/bash
# certification of HEAD: every GPU test, smoke, default bench x2, reference arm
cd "$(dirname "$0")/../../.."
O=gpurun_out/fe; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py > $O/bench2.json 2> $O/bench2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
tail -2 $O/pytest_gpu.txt; tail -1 $O/smoke.txt; head -c 300 $O/bench.json
