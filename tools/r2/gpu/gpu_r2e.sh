#!/bin/bash
# round 2: predicated-remainder SpMM + papers-q shape sweep (ld4 = 12: G, NC, U, min blocks/SM), Reddit check
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_train_sparse.py > gpurun_out/r2e_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2e_pytest.txt
for sh in default 16,1,8,3 16,1,16,2 16,1,16,3; do
  if [ $sh = default ]; then unset PGCN_SPMM_TABLE; else export PGCN_SPMM_TABLE="12=$sh"; fi
  timeout 900 python bench.py --config papers-q --no-cpu --no-e2e --no-ablation --steps 5 > gpurun_out/r2e_papers_$sh.json 2> gpurun_out/r2e_papers_$sh.err
done
unset PGCN_SPMM_TABLE
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/r2e_bench_reddit.json 2> gpurun_out/r2e_bench_reddit.err
tail -2 gpurun_out/r2e_pytest.txt
timeout 600 python bench.py --no-cpu --no-e2e --transport push > gpurun_out/r2e_bench_reddit_push.json 2> gpurun_out/r2e_bench_reddit_push.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2e_papers_e_launches.csv python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2e_ncu_papers_e.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_bwd|k_umma_gemm" --launch-skip 60 --launch-count 8 -o gpurun_out/r2e_papers_e_full python bench.py --config papers-e --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2e_ncu_papers_e_full.log 2>&1
