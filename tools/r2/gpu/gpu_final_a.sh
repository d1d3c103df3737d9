#!/bin/bash
# round-2 final evidence, part A: GPU tests, smoke, the default bench (twice) + reference arm, ncu launch list of
# the default bench and full captures of its top kernels (exported to CSV on the box)
cd "$(dirname "$0")/../../.."
O=gpurun_out/fa; mkdir -p $O
nvidia-smi -L > $O/gpu.txt; nproc >> $O/gpu.txt; free -g >> $O/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py > $O/bench2.json 2> $O/bench2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $O/reddit_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_reddit.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_tc|k_umma_gemm|k_spmm_bwd|k_dropout|k_split_bf16" --launch-skip 400 --launch-count 14 -o /tmp/fa_reddit python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_reddit_full.log 2>&1
ncu -i /tmp/fa_reddit.ncu-rep --page raw --csv > $O/reddit_full_raw.csv 2>/dev/null
cp /tmp/fa_reddit.ncu-rep $O/ 2>/dev/null
tail -2 $O/pytest_gpu.txt; tail -1 $O/smoke.txt; head -c 600 $O/bench.json
