for C in products yelp; do
B="python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv $B > /dev/null 2>&1
echo "== $C"
python tools/launch_table.py gpurun_out/launches_$C.csv 120 | head -16
done
