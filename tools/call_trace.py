#!/usr/bin/env python
"""Kernel-level device trace of one device-pointer emm call (GPU tool, not a
test): every launch of the call with its start offset, duration and the gap
before it, from CUPTI via torch.profiler; L2 flushed before each rep.

    python tools/call_trace.py --shape 1531,997,2049,N,N [--math 3xtf32] [--pad 13,7,5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1531,997,2049,N,N")
    ap.add_argument("--math", default="3xtf32")
    ap.add_argument("--pad", default="0,0,0")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    M, N, K, tA, tB = a.shape.split(",")
    M, N, K = int(M), int(N), int(K)
    pa, pb, pc = (int(x) for x in a.pad.split(","))
    dev = torch.device("cuda", 0)
    ra, ca = (M, K) if tA == "N" else (K, M)
    rb, cb = (K, N) if tB == "N" else (N, K)
    lda, ldb, ldc = ra + pa, rb + pb, M + pc
    A = torch.rand(ca * lda, device=dev)
    B = torch.rand(cb * ldb, device=dev)
    C = torch.zeros(N * ldc, device=dev)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, device=dev)
    s = torch.cuda.current_stream(dev)

    def call():
        st = emm.sgemm_ptr(tA, tB, M, N, K, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0, C.data_ptr(), ldc,
                           s.cuda_stream, a.math)
        assert st == 0, emm.strerror(st)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            flush.fill_(1.0)
            call()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    # group: a call = the launches after each fill kernel
    calls, cur = [], None
    for e in ev:
        if "fill" in e.name.lower() or "FillFunctor" in e.name:
            cur = {"flush_end": e.time_range.end, "k": []}
            calls.append(cur)
        elif cur is not None:
            cur["k"].append(e)
    print(f"{M}x{N}x{K} {tA}{tB} {a.math} pad {a.pad}")
    for i, c in enumerate(calls):
        t0 = c["flush_end"]
        prev = t0
        tot = (c["k"][-1].time_range.end - t0) if c["k"] else 0
        print(f" call {i}: flush end -> last kernel end {tot:.1f} us")
        for e in c["k"]:
            st, en = e.time_range.start, e.time_range.end
            print(f"   +{st - t0:7.1f} us  gap {st - prev:6.1f}  dur {en - st:7.1f}  {e.name[:90]}")
            prev = en


if __name__ == "__main__":
    main()
