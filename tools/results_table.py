#!/usr/bin/env python
"""Render BASELINE.md §5 rows from a bench_sweep.py JSONL file and a bench.py
JSON line (both committed under profiles/)."""
import json
import sys


def main(sweep, bench=None):
    print("| Config | Path | GPUs | Median time | GFLOP/s | % roofline (peak) | GB/s compulsory | back-to-back (graph, no flush) |")
    print("|---|---|---|---|---|---|---|---|")
    for line in open(sweep):
        r = json.loads(line)
        t = r["median_ms"] * 1e3
        ts = f"{t:.1f} µs" if t < 1000 else f"{t / 1e3:.3f} ms"
        print(f"| {r['config']} {r['M']}×{r['N']}×{r['K']} {r['transA']}{r['transB']} | {r['math']} | 1 | {ts} | "
              f"{r['gflops']:.0f} | {r['pct_roofline']:.1f} ({r['roofline_tflops']:.0f} TF) | {r['gbs']:.0f} | "
              + (f"{r['b2b_graph_us']:.1f} µs |" if r.get('b2b_graph_us') else "— |"))
    if bench:
        d = json.loads(open(bench).read().strip().splitlines()[-1])
        rf = d["roofline"]
        print(f"\nbench.py (c5 32768³ NN, {d['config']['math']}): {d['value']:.0f} GFLOP/s per step "
              f"({d['ms_per_step']:.1f} ms), kernel {rf['achieved']:.1f} TFLOP/s = {rf['frac']:.3f} of the "
              f"sustained-derived peak ({rf['peak']:.1f}) / {rf['frac_burst']:.3f} of burst ({rf['peak_burst']:.1f}); "
              f"clocks {d['clocks']}")


if __name__ == "__main__":
    main(*sys.argv[1:])
