#!/bin/bash
# round 2: PUSH transport tests + sanitizer, transports A/B on Reddit, papers-q bench + ncu, gather ceiling
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -s -p no:cacheprovider tests/test_gpu_exchange.py "tests/test_gpu_fullsize_step.py::test_full_size_two_iterations[products]" tests/test_gpu_gemm.py -k "exchange or products or full_size" > gpurun_out/r2d_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.txt
for T in memcheck racecheck; do
  echo "== $T" >> gpurun_out/r2d_sanitizer.txt
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/r2/sanitize_exchange.py >> gpurun_out/r2d_sanitizer.txt 2>&1
done
timeout 600 python tools/r2/gather_ceiling.py > gpurun_out/r2d_gather_ceiling.jsonl 2> gpurun_out/r2d_gather_ceiling.err
for tr in push loopback local; do timeout 600 python bench.py --no-cpu --no-e2e --transport $tr > gpurun_out/r2d_bench_reddit_$tr.json 2> gpurun_out/r2d_bench_reddit_$tr.err; done
timeout 600 python bench.py --no-cpu --no-e2e --mode vanilla > gpurun_out/r2d_bench_reddit_vanilla.json 2> gpurun_out/r2d_bench_reddit_vanilla.err
timeout 1200 python bench.py --config papers-q --no-cpu --steps 10 > gpurun_out/r2d_bench_papers.json 2> gpurun_out/r2d_bench_papers.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2d_papers_launches.csv python bench.py --config papers-q --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2d_ncu_papers.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_bwd|k_umma_gemm" --launch-skip 60 --launch-count 8 -o gpurun_out/r2d_papers_full python bench.py --config papers-q --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2d_ncu_papers_full.log 2>&1
tail -2 gpurun_out/r2d_pytest.txt
