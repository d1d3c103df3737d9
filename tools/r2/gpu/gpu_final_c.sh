#!/bin/bash
# round-2 final evidence of HEAD (after the BK16 GEMM change): GPU tests, smoke, default bench x2, reference arm,
# every config, ncu launch list of the default bench
cd "$(dirname "$0")/../../.."
O=gpurun_out/${FINAL_DIR:-fc}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py > $O/bench2.json 2> $O/bench2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
bash tools/r2/all_configs.sh $O/all
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $O/reddit_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_reddit.log 2>&1
tail -2 $O/pytest_gpu.txt; tail -1 $O/smoke.txt; head -c 300 $O/bench.json
