"""Host-side workload build of one rank of the papers100M-shaped multi-GPU run (bench.py's
build_rank_workload: the full synthetic structure generated and partitioned on the rank, inputs only for the
rank's own rows), timed with its peak resident memory -- no GPU needed.  Without a process group the
train count is the rank's own (the bench all-reduces it).

    python tools/r2/papers_rank_build.py [--parts 8] [--rank 0]
"""
import argparse
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--config", default="papers")
    a = ap.parse_args()
    import bench
    from paper_2203_10428_b200 import pgcn
    t0 = time.time()
    g, m, _, part, t_build = bench.build_rank_workload(a.config, a.parts, a.rank, None, pgcn)
    v = part.view(a.rank)
    print(json.dumps({"config": a.config, "n": g.n, "nnz": g.nnz, "parts": a.parts, "rank": a.rank,
                      "build_s": t_build, "wall_s": time.time() - t0,
                      "peak_rss_GB": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
                      "rank_rows": int(v["n_inner"]), "rank_X_GB": g.X.nbytes / 1e9,
                      "threads": len(os.sched_getaffinity(0))}))


if __name__ == "__main__":
    main()
