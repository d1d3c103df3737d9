"""Writes the round-2 results table of BASELINE.md (between the r2-table markers) and
profiles/r2_all_configs.md from a directory of bench.py JSON lines (tools/r2/all_configs.sh output).
python tools/r2/baseline_table.py gpurun_out/r2_all"""
import json
import os
import sys

ROWS = [
    ("reddit_pipe", "Reddit-shaped (233K, 113.6M nnz, 602-256×3-41)", "fp32", "PIPE / loopback"),
    ("reddit_pipe_local", "Reddit-shaped", "fp32", "PIPE / local"),
    ("reddit_pipe_push", "Reddit-shaped", "fp32", "PIPE / push (N2)"),
    ("reddit_vanilla", "Reddit-shaped", "fp32", "VANILLA / loopback"),
    ("reddit_pipe_gf", "Reddit-shaped", "fp32", "PIPE-GF / loopback"),
    ("reddit_depth2", "Reddit-shaped", "fp32", "PIPE depth 2 / loopback"),
    ("reddit_pipe_bf16payload", "Reddit-shaped", "fp32 + bf16 payloads (N1(iv))", "PIPE / loopback"),
    ("reddit_notiles", "Reddit-shaped", "fp32, gather-only (IEEE fp32 sums)", "PIPE / loopback"),
    ("reddit_gcn", "Reddit-shaped, GCN-sym (N3)", "fp32", "PIPE / loopback"),
    ("reddit_bf16gather", "Reddit-shaped", "bf16 gather", "PIPE / loopback"),
    ("reddit_bf16all", "Reddit-shaped", "bf16 gather + bf16 GEMM", "PIPE / loopback"),
    ("reddit_lean", "Reddit-shaped, lean-memory mode (N1(iii))", "fp32", "PIPE / loopback"),
    ("products_pipe", "products-shaped (2.45M, 61.8M nnz, 100-128-128-47)", "fp32", "PIPE / loopback"),
    ("products_bf16gather", "products-shaped", "bf16 gather", "PIPE / loopback"),
    ("yelp_pipe_gf", "Yelp-shaped (717K, 7.0M nnz, 300-512×3-100, BCE)", "fp32", "PIPE-GF / loopback"),
    ("yelp_bf16all_gf", "Yelp-shaped", "bf16 gather + bf16 GEMM", "PIPE-GF / loopback"),
    ("papers_q", "papers-q (papers100M recipe at ¼: 27.8M, 404M nnz, 128-48-48-172)", "fp32", "PIPE / %s"),
    ("papers_q_lean", "papers-q, lean-memory mode (N1(iii))", "fp32", "PIPE / %s"),
    ("cora_pipe", "Cora-shaped (2.7K, 10.6K nnz, 1433-16-7)", "fp32", "PIPE / loopback"),
]


def main():
    src = sys.argv[1]
    out = ["| config | tier | mode / transport | ep/s | ms/epoch | dominant kernel (ms/step): roofline frac | "
           "aggregation: B_min/HBM frac | exposed comm ms | e2e ep/s |",
           "|---|---|---|---|---|---|---|---|---|"]
    for name, cfg, tier, mode in ROWS:
        p = os.path.join(src, name + ".json")
        if not os.path.exists(p):
            continue
        try:
            d = json.loads(open(p).read().strip().splitlines()[-1])
        except Exception:
            continue
        exp = d["comm"] and d["comm"].get("exposed_ms_per_step")
        r = d["roofline"]
        ra = d.get("roofline_aggregation")
        ms_k = d["kernels"][r["kernel"]]["ms_per_step"] if "kernels" in d else d["breakdown"][r["kernel"]]["ms_per_step"]
        if "%s" in mode:
            mode = mode % d["config"].get("transport")
        out.append("| %s | %s | %s | %.2f | %.2f | %s (%.2f): %s %.3f | %s | %s | %s |" % (
            cfg, tier, mode, d["value"], d["ms_per_step"], r["kernel"], ms_k, r["bound"], r["frac"],
            ("%.3f" % ra["frac"]) if ra else "—",
            ("%.2f" % exp) if exp is not None else "—", ("%.2f" % d["e2e"]["value"]) if d.get("e2e") else "—"))
    ref = os.path.join(src, "reference_reddit.json")
    if os.path.exists(ref):
        try:
            d = json.loads(open(ref).read().strip().splitlines()[-1])
            out.append("")
            out.append("Reference arm (`bench.py --impl reference`, the fp64 oracle on %d host cores): %.4g ep/s (%s)." % (
                d["cpu_baseline"]["cores"], d["value"], d["cpu_baseline"]["sample"]))
        except Exception:
            pass
    table = "\n".join(out)
    open(os.path.join("profiles", "r2_all_configs.md"), "w").write(
        "# r2: every config / tier / mode (bench.py lines in %s)\n\n%s\n" % (src, table))
    s = open("BASELINE.md").read()
    a, b = s.index("<!-- r2-table begin -->"), s.index("<!-- r2-table end -->")
    s = s[:a] + "<!-- r2-table begin -->\n" + table + "\n" + s[b:]
    open("BASELINE.md", "w").write(s)


if __name__ == "__main__":
    main()
