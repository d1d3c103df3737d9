#!/bin/bash
# round 2: every config / tier / mode of the BASELINE.md table, one bench.py line each (+ the reference arm)
cd "$(dirname "$0")/../.."
D=${1:-gpurun_out/r2_all}
mkdir -p $D
run() { name=$1; shift; timeout 1200 python bench.py --no-cpu "$@" > $D/$name.json 2> $D/$name.err; }
run reddit_pipe
run reddit_pipe_gf --smooth gf --no-e2e
run reddit_vanilla --mode vanilla --no-e2e
run reddit_pipe_local --transport local --no-e2e
run reddit_pipe_push --transport push --no-e2e
run reddit_pipe_bf16payload --halo-payload bf16 --no-e2e
run reddit_notiles --no-tiles --no-e2e
run reddit_gcn --model gcn --no-e2e
run reddit_bf16gather --gather bf16 --no-e2e
run reddit_bf16all --gather bf16 --gemm bf16 --no-e2e
run reddit_depth2 --depth 2 --no-e2e
run reddit_lean --lean --no-e2e
run products_pipe --config products --no-e2e
run products_bf16gather --config products --gather bf16 --no-e2e
run yelp_pipe_gf --config yelp --smooth gf --no-e2e
run yelp_bf16all_gf --config yelp --smooth gf --gather bf16 --gemm bf16 --no-e2e
run cora_pipe --config cora --no-e2e
run papers_q --config papers-q --steps 10
run papers_q_lean --config papers-q --lean --steps 10
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $D/reference_reddit.json 2> $D/reference_reddit.err
ls $D | wc -l
