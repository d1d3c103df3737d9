"""Per-launch table of the 26 tcgen05 GEMM launches of one Reddit step (tools/prof_gemm.sh output)."""
import collections
import csv
import sys

NAMES = ["fwd l1 T p0", "fwd l1 self p0", "fwd l1 T p1", "fwd l1 self p1", "fwd l2 p0", "fwd l2 p1", "fwd l3 p0",
         "fwd l3 p1", "fwd l4 T p0", "fwd l4 self p0", "fwd l4 T p1", "fwd l4 self p1", "dw l4 p0", "J l4 p0",
         "dw l4 p1", "J l4 p1", "dw l3 p0", "da l3 p0", "dw l3 p1", "da l3 p1", "dw l2 p0", "da l2 p0", "dw l2 p1",
         "da l2 p1", "dw l1 p0", "dw l1 p1"]
SC = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}


def main(path):
    hdr, d = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        x = dict(zip(hdr, r))
        d.setdefault(int(x["ID"]), {})[x["Metric Name"]] = (x["Metric Value"].replace(",", ""), x["Metric Unit"])
    tot = 0.0
    print("| launch | ms | tensor % | SM % | DRAM MB | L2 MB |\n|---|---|---|---|---|---|")
    for n, v in zip(NAMES, d.values()):
        t = float(v["gpu__time_duration.sum"][0]) * SC.get(v["gpu__time_duration.sum"][1], 1.0)
        tot += t
        g = lambda k: v.get(k, ("nan", ""))[0]  # noqa: E731
        print("| %s | %.3f | %s | %s | %.0f | %.0f |" % (
            n, t, g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            (float(g("dram__bytes_read.sum")) + float(g("dram__bytes_write.sum"))) / 1e6, float(g("lts__t_bytes.sum")) / 1e6))
    print("| total | %.3f | | | | |" % tot)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_launches.csv")
