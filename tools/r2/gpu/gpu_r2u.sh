#!/bin/bash
# L2 persisting window over the gathered table of the gather SpMMs (PGCN_L2_PERSIST_MB) A/B
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2u; mkdir -p $O
python -c "
import torch
p=torch.cuda.get_device_properties(0)
print('l2', p.L2_cache_size/2**20, 'MB')" > $O/dev.txt 2>&1
for mb in 0 48 80 112; do
  PGCN_L2_PERSIST_MB=$mb timeout 900 python bench.py --no-cpu --no-e2e --no-ablation --steps 20 > $O/reddit_l2p$mb.json 2> $O/reddit_l2p$mb.err
done
for mb in 0 80; do
  PGCN_L2_PERSIST_MB=$mb timeout 900 python bench.py --config products --no-cpu --no-e2e --no-ablation --steps 10 > $O/products_l2p$mb.json 2> $O/products_l2p$mb.err
  PGCN_L2_PERSIST_MB=$mb timeout 900 python bench.py --config papers-q --no-cpu --no-e2e --no-ablation --steps 10 > $O/papersq_l2p$mb.json 2> $O/papersq_l2p$mb.err
done
ls $O
