#!/bin/bash
# round 2, first GPU pass: all GPU tests, then the bench in its default (loopback) and two variants
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.txt
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "rc=$?" >> gpurun_out/r2a_bench.err
timeout 400 python bench.py --transport local --no-cpu --no-e2e > gpurun_out/r2a_bench_local.json 2> gpurun_out/r2a_bench_local.err
timeout 400 python bench.py --mode vanilla --no-cpu --no-e2e > gpurun_out/r2a_bench_vanilla.json 2> gpurun_out/r2a_bench_vanilla.err
tail -3 gpurun_out/r2a_pytest.txt
