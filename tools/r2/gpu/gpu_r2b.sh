#!/bin/bash
# round 2, second GPU pass: GPU tests (incl. exchange, full-size step parity, large dW), sanitizer on the
# loopback exchange, three bench runs (mode study), launch list and full ncu captures of the top kernels
cd "$(dirname "$0")/../../.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2b_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.txt
for T in memcheck racecheck synccheck; do
  echo "== $T" >> gpurun_out/r2b_sanitizer.txt
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/r2/sanitize_exchange.py >> gpurun_out/r2b_sanitizer.txt 2>&1
done
for k in 1 2 3; do timeout 600 python bench.py --no-cpu > gpurun_out/r2b_bench_$k.json 2> gpurun_out/r2b_bench_$k.err; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2b_ncu_bench.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_spmm_fwd|k_spmm_tc|k_umma_gemm|k_spmm_bwd|k_dropout" --launch-skip 300 --launch-count 12 -o gpurun_out/r2b_full python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r2b_ncu_full.log 2>&1
tail -3 gpurun_out/r2b_pytest.txt
