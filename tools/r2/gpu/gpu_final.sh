#!/bin/bash
# round 2 final evidence pass: GPU tests, smoke, sanitizers, the default bench + reference arm, ncu launch
# lists and full captures (exported to CSV on the box), all configs for BASELINE.md
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
for T in memcheck racecheck synccheck; do
  echo "== $T exchange" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/r2/sanitize_exchange.py >> $O/sanitizer.txt 2>&1
  echo "== $T engine" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize.py >> $O/sanitizer.txt 2>&1
  echo "== $T tiles" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_tiles.py >> $O/sanitizer.txt 2>&1
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py > $O/bench2.json 2> $O/bench2.err
timeout 1200 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $O/reddit_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_reddit.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_tc|k_umma_gemm|k_spmm_bwd|k_dropout|k_split_bf16|k_grad_reduce" --launch-skip 380 --launch-count 16 -o /tmp/final_reddit python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_reddit_full.log 2>&1
ncu -i /tmp/final_reddit.ncu-rep --page raw --csv > $O/reddit_full_raw.csv 2>/dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --launch-skip 200 --launch-count 160 --csv --log-file $O/papers_e_launches.csv python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_papers_e.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file $O/products_launches.csv python bench.py --config products --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_products.log 2>&1
rm -rf gpurun_out/r2_all
bash tools/r2/all_configs.sh
du -sh gpurun_out
