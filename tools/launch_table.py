"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum launch list (last step's launches)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
tail = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[ii], {"k": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
L = list(launch.values())
if tail:
    L = L[-tail:]
tot = collections.defaultdict(float)
cnt = collections.Counter()
dram = collections.defaultdict(float)
for d in L:
    k = d["k"].split("(")[0]
    tot[k] += d["gpu__time_duration.sum"]
    cnt[k] += 1
    dram[k] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
T = sum(tot.values())
print("%d launches, %.3f ms" % (len(L), T / 1e6))
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print("%-70s %4d %8.3f ms %5.1f%%  %.3f ms/launch  %.0f MB/launch" % (k[:70], cnt[k], v / 1e6, 100 * v / T, v / 1e6 / cnt[k],
                                                                   dram[k] / 1e6 / cnt[k]))
