"""Random-row gather ceiling on this B200 (roofline denominator of the DRAM-served aggregation):
pgcn_dev_gather_read over a ~6 GB table (far beyond the 126 MB L2) with uniformly random row ids, for
the row widths of the workloads (48 floats: papers100M hidden, 128: products, 256: Reddit hidden).
Prints one JSON line per width: useful row bytes / time (GB/s) and the fraction of the HBM copy peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
L = pgcn.lib()
st = torch.cuda.current_stream()
out = torch.empty(148 * 8 * 256 * 2, device="cuda")
g = torch.Generator(device="cuda").manual_seed(7)
for F in (48, 128, 256):
    rows = (6 << 30) // (4 * F)
    tab = torch.randn(rows, F, device="cuda", generator=g)
    n_idx = 100_000_000 if F <= 128 else 25_000_000
    idx = torch.randint(0, rows, (n_idx,), device="cuda", dtype=torch.int32, generator=g)
    best = {}
    for variant in (0, 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        rc = L.pgcn_dev_gather_read(tab.data_ptr(), F, idx.data_ptr(), n_idx, out.data_ptr(), variant, st.cuda_stream)
        assert rc == 0, rc
        e0.record()
        for _ in range(3):
            L.pgcn_dev_gather_read(tab.data_ptr(), F, idx.data_ptr(), n_idx, out.data_ptr(), variant, st.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        best[variant] = 3 * n_idx * 4 * F / (e0.elapsed_time(e1) / 1e3) / 1e9
    v = max(best.values())
    print(json.dumps({"row_floats": F, "row_bytes": 4 * F, "table_GB": rows * F * 4 / 1e9, "n_idx": n_idx,
                      "gather_GBps": v, "hbm_peak_GBps": peak, "frac_of_hbm": v / peak,
                      "per_variant": best}))
    del tab, idx
