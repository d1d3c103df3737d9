B="python bench.py --config papers-q --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_papers.csv $B > gpurun_out/papers_ncu.log 2>&1
echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/launches_papers.csv 200 | head -30
