#!/usr/bin/env python
"""A/B table from bench_sweep.py --variants output files: per config, the
median time of each variant and the ratio to the first one."""
import json
import sys


def main(paths):
    rows = [json.loads(l) for p in paths for l in open(p)]
    by, order = {}, []
    for r in rows:
        key = (r["config"], r["math"])
        if key not in by:
            by[key] = {}
            order.append(key)
        by[key][r.get("variant", "")] = r
    variants = []
    for r in rows:
        if r.get("variant", "") not in variants:
            variants.append(r.get("variant", ""))
    print("| config | math | " + " | ".join(f"{v} (us, TFLOP/s)" for v in variants) + " | ratio |")
    print("|---|---|" + "---|" * (len(variants) + 1))
    for key in order:
        d = by[key]
        cells = []
        for v in variants:
            r = d.get(v)
            cells.append(f"{r['median_ms'] * 1e3:.1f}, {r['gflops'] / 1e3:.1f}" if r else "-")
        base = d.get(variants[0])
        last = d.get(variants[-1])
        ratio = f"{base['median_ms'] / last['median_ms']:.3f}" if base and last else "-"
        print(f"| {key[0]} | {key[1]} | " + " | ".join(cells) + f" | {ratio} |")


if __name__ == "__main__":
    main(sys.argv[1:])
