#!/bin/bash
# column-chunk count A/B for the L2-chunked gathers (Reddit-shaped: 238 MB forward / 119 MB transposed tables)
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2q; mkdir -p $O
for rep in 1 2; do
for nch in 2 3 4; do
  PGCN_SPMM_NCH=$nch timeout 600 python bench.py --no-cpu --no-e2e --no-ablation --steps 30 > $O/reddit_nch${nch}_$rep.json 2> $O/reddit_nch${nch}_$rep.err
done
done
PGCN_SPMM_NCH=4 PGCN_SPMM_L2MB=64 timeout 600 python bench.py --no-cpu --no-e2e --no-ablation --steps 30 > $O/reddit_nch4_l2mb64.json 2> $O/reddit_nch4_l2mb64.err
for nch in 2 4; do
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $O/launches_nch$nch.csv env PGCN_SPMM_NCH=$nch python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu_nch$nch.log 2>&1
done
ls $O
