#!/usr/bin/env python
"""Per-launch time breakdown of one emm_sgemm_ex call (GPU tool, not a test).

For each shape: median device time of the whole call (L2 flushed before each
rep), and the same call with the library's per-launch profiling on (events
around every launch: GEMM launches vs the rest — split pass, split-K reduce).

    python tools/breakdown.py [--shapes 1024,1024,1024,N,N;1531,997,2049,N,N] [--maths 3xtf32,1xtf32]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402

DEFAULT = "1000,1000,1000,N,N;1024,1024,1024,N,N;2048,2048,2048,N,N;1531,997,2049,N,N;4096,4096,4096,N,N"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--maths", default="3xtf32,1xtf32")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    for spec in args.shapes.split(";"):
        M, N, K, tA, tB = spec.split(",")
        M, N, K = int(M), int(N), int(K)
        ra, ca = (M, K) if tA == "N" else (K, M)
        rb, cb = (K, N) if tB == "N" else (N, K)
        A = torch.rand(ca, ra, device=dev, generator=g).t()
        B = torch.rand(cb, rb, device=dev, generator=g).t()
        C = torch.zeros(N, M, device=dev).t()
        for math in args.maths.split(","):
            ws = torch.empty(emm.workspace_bytes(tA, tB, M, N, K, math), dtype=torch.uint8, device=dev)
            call = lambda: emm.sgemm_ex(A, B, C, 1.0, 0.0, tA, tB, math=math, workspace=ws)  # noqa: E731
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            tot = []
            for _ in range(args.reps):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                torch.cuda.synchronize()
                tot.append(e0.elapsed_time(e1))
            emm.profile_read()
            emm.profile_enable(True)
            gm, om = [], []
            for _ in range(args.reps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                call()
                torch.cuda.synchronize()
                a, an, b, bn = emm.profile_read()
                gm.append(a)
                om.append(b)
            emm.profile_enable(False)
            # warm back-to-back: 50 calls, no flush
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(50):
                call()
            e1.record()
            torch.cuda.synchronize()
            warm = e0.elapsed_time(e1) / 50
            print(json.dumps({"M": M, "N": N, "K": K, "tA": tA, "tB": tB, "math": math,
                              "call_ms": statistics.median(tot), "gemm_ms": statistics.median(gm),
                              "other_ms": statistics.median(om), "launches": int(an + bn),
                              "warm_b2b_ms": warm,
                              "tflops_call": 2 * M * N * K / statistics.median(tot) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
