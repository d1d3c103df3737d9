#!/bin/bash
# ncu --set full of the papers-e shape's top kernels with HEAD (GEMMs after the k-block / dW-plan changes)
cd "$(dirname "$0")/../../.."
O=gpurun_out/r2z; mkdir -p $O
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_umma_gemm|k_spmm_fwd|k_spmm_bwd" --launch-skip 120 --launch-count 14 -o /tmp/r2z_papers_e python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > $O/ncu.log 2>&1
ncu -i /tmp/r2z_papers_e.ncu-rep --page raw --csv > $O/papers_e_full_raw.csv 2>/dev/null
timeout 900 python bench.py --config papers-e --no-cpu --no-e2e --no-ablation --steps 10 > $O/papers_e.json 2> $O/papers_e.err
ls -la $O
