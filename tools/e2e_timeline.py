#!/usr/bin/env python
"""Device timeline of one emm_sgemm_host call (GPU tool, not a test): runs the
host-buffer entry under torch.profiler (CUPTI sees the library's own streams)
and reports when the first GEMM starts, GPU idle time between kernels, the
H2D / D2H copy spans and the exposed tail after the last kernel.

    python tools/e2e_timeline.py [--n 32768] [--math 3xtf32]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--math", default="3xtf32")
    args = ap.parse_args()
    n = args.n
    g = torch.Generator().manual_seed(0)
    hA = (torch.rand(n * n, generator=g) * 2 - 1).pin_memory()
    hB = (torch.rand(n * n, generator=g) * 2 - 1).pin_memory()
    hC = torch.empty(n * n).pin_memory()
    emm.sgemm_host("N", "N", n, n, n, 1.0, hA, n, hB, n, 0.0, hC, n, math=args.math)   # warm (allocations)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        emm.sgemm_host("N", "N", n, n, n, 1.0, hA, n, hB, n, 0.0, hC, n, math=args.math)
        wall = time.perf_counter() - t0
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev if "Memcpy" not in e.name
                   and "Memset" not in e.name], key=lambda x: x[0])
    cpy = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev if "Memcpy" in e.name],
                 key=lambda x: x[0])
    t_first = min([k[0] for k in kern] + [c[0] for c in cpy])
    t_last = max([k[1] for k in kern] + [c[1] for c in cpy])
    gemm = [k for k in kern if "sgemm" in k[2] or "tc1w" in k[2] or "tc_xs" in k[2]]
    busy, last_end = 0.0, None
    for s, e, _ in kern:   # union of kernel intervals
        if last_end is None or s >= last_end:
            busy += e - s
            last_end = e
        elif e > last_end:
            busy += e - last_end
            last_end = e
    h2d = [c for c in cpy if "HtoD" in c[2]]
    d2h = [c for c in cpy if "DtoH" in c[2]]
    out = {
        "n": n, "math": args.math, "wall_ms": wall * 1e3, "span_ms": (t_last - t_first) / 1e3,
        "first_gemm_start_ms": (gemm[0][0] - t_first) / 1e3 if gemm else None,
        "kernel_busy_ms": busy / 1e3, "kernels": len(kern), "gemms": len(gemm),
        "h2d_span_ms": ((h2d[-1][1] - h2d[0][0]) / 1e3) if h2d else None,
        "h2d_busy_ms": sum(e - s for s, e, _ in h2d) / 1e3,
        "d2h_busy_ms": sum(e - s for s, e, _ in d2h) / 1e3,
        "tail_after_last_kernel_ms": (t_last - max(k[1] for k in kern)) / 1e3,
        "gflops_span": 2.0 * n ** 3 / ((t_last - t_first) * 1e-6) / 1e9,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
