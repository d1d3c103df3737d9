#!/bin/bash
# round 2: papers-q shape (the north_star flagship per-GPU shape) -- bench, launch list with DRAM bytes,
# full ncu capture of the aggregation kernels, and the random-row gather ceiling
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
for K in 0 1024 256 64; do PGCN_DW_KMAX=$K timeout 600 python tools/r2/dw_chain.py >> gpurun_out/r2c_dw_chain.jsonl 2>> gpurun_out/r2c_dw_chain.err; done
timeout 600 python tools/r2/gather_ceiling.py > gpurun_out/r2c_gather_ceiling.jsonl 2> gpurun_out/r2c_gather_ceiling.err
timeout 1200 python bench.py --config papers-q --no-cpu --steps 10 > gpurun_out/r2c_bench_papers.json 2> gpurun_out/r2c_bench_papers.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2c_papers_launches.csv python bench.py --config papers-q --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2c_ncu_papers.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_bwd|k_umma_gemm" --launch-skip 60 --launch-count 8 -o gpurun_out/r2c_papers_full python bench.py --config papers-q --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2c_ncu_papers_full.log 2>&1
ls -la gpurun_out | tail -5
timeout 1800 python -m pytest -q -s -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_fullsize_step.py tests/test_gpu_exchange.py tests/test_gpu_parity.py tests/test_gpu_bf16_gather.py tests/test_gpu_gcn.py > gpurun_out/r2c_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.txt
for k in 1 2; do timeout 600 python bench.py --no-cpu > gpurun_out/r2c_bench_reddit_$k.json 2> gpurun_out/r2c_bench_reddit_$k.err; done
tail -2 gpurun_out/r2c_pytest.txt
