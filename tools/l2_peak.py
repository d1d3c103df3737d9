"""L2 read-bandwidth microbenchmark variants (pgcn_dev_l2_read) at several buffer sizes (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402

L = pgcn.lib()
s = torch.cuda.current_stream().cuda_stream
out = torch.empty(148 * 8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mb in (16, 32, 64, 96):
    nbytes = mb << 20
    buf = torch.ones(nbytes // 4, device="cuda")
    row = []
    for v in (0, 1, 2):
        reps = 50
        L.pgcn_dev_l2_read(buf.data_ptr(), nbytes, (v << 24) | 2, out.data_ptr(), s)
        e0.record()
        L.pgcn_dev_l2_read(buf.data_ptr(), nbytes, (v << 24) | reps, out.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        row.append(nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print("%3d MB: " % mb + "  ".join("v%d %.0f GB/s" % (i, x) for i, x in enumerate(row)), flush=True)
