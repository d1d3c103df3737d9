#!/bin/bash
# round 2: Reddit last-layer variants (train-sparse gather vs all-row tile path; 44-wide row shapes), papers-q shape
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py --no-cpu --no-e2e --no-ablation "$@" > gpurun_out/r2i_$name.json 2> gpurun_out/r2i_$name.err; }
run reddit_default
run reddit_notrainsparse --no-train-sparse
PGCN_SPMM_TABLE="11=8,2,4,3" run reddit_w11_8243
PGCN_SPMM_TABLE="11=4,3,4,3" run reddit_w11_4343
PGCN_SPMM_TABLE="11=16,1,8,3" run reddit_w11_16183
PGCN_SPMM_TABLE="12=8,2,4,3" run papersq_w12_8243 --config papers-q --steps 5
run papersq_default --config papers-q --steps 5
