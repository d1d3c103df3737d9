B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --gather bf16 --gemm bf16"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bf16gemm.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_bf16gemm.csv 110 2>/dev/null | head -12
python3 - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/launches_bf16gemm.csv')))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    d = launch.setdefault(r[ii], {"k": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
L = list(launch.values())
idx = [i for i, d in enumerate(L) if "k_opt" in d["k"]]
for j, d in enumerate(L[idx[-2] + 1: idx[-1] + 1]):
    if "umma" in d["k"] or "colsum" in d["k"]:
        print(j, "%-35s %.3f ms %6.0f MB" % (d["k"][:35], d["gpu__time_duration.sum"] / 1e6, (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e6))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 104 -c 1 -o gpurun_out/bf16_dw $B > /dev/null 2>&1
