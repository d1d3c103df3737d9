#!/bin/bash
# round-2 final evidence, part B: every config of BASELINE.md, ncu launch lists of papers-e and products,
# compute-sanitizer on the exchange transports and the lean mode
cd "$(dirname "$0")/../../.."
O=gpurun_out/fb; mkdir -p $O
bash tools/r2/all_configs.sh $O/all
for cfg in reddit yelp; do
  PGCN_TC_BNMAX=128 timeout 900 python bench.py --config $cfg --no-cpu --no-e2e --no-ablation > $O/${cfg}_bn128.json 2> $O/${cfg}_bn128.err
done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --launch-skip 200 --launch-count 160 --csv --log-file $O/papers_e_launches.csv python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_papers_e.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file $O/products_launches.csv python bench.py --config products --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_products.log 2>&1
for T in memcheck racecheck synccheck; do
  echo "== $T exchange + lean" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/r2/sanitize_exchange.py >> $O/sanitizer.txt 2>&1
done
du -sh gpurun_out
