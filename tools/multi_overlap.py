#!/usr/bin/env python
"""GPU tool (not a test): does the row-sharded path overlap B's transfer with
the panel GEMMs?  P virtual ranks on one GPU (emm_debug_comm_create_local; the
copy-engine ring of DESIGN.md §7 with events in place of flags) run one
emm_sgemm_multi under torch.profiler (CUPTI); for every rank's device-to-device
chunk copies the tool reports how much of their time overlaps a GEMM kernel
(of any rank) and how long each rank's compute stream waited before its first
panel GEMM.  One GPU shares its HBM and SMs between the virtual ranks, so the
times are not multi-GPU times; the concurrency is the point.

    python tools/multi_overlap.py [--P 2] [--n 8192]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import datagen  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402


def overlap(iv, others):
    s, e = iv
    tot = 0.0
    for a, b in others:
        lo, hi = max(s, a), min(e, b)
        if hi > lo:
            tot += hi - lo
    return min(tot, e - s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--n", type=int, default=8192)
    a = ap.parse_args()
    P, n = a.P, a.n
    dev = torch.device("cuda", 0)
    comms = emm.local_comms(P)
    streams = [torch.cuda.Stream(dev) for _ in range(P)]
    Bsrc = datagen.matrix("uniform", datagen.TAG_B, n, n, device=dev)
    ranks = []
    for r, c in enumerate(comms):
        r0, rows = emm.row_partition(n, P, r)
        A = datagen.submatrix("uniform", datagen.TAG_A, n, n, torch.arange(r0, r0 + rows), device=dev)
        B = Bsrc.clone() if r == 0 else torch.zeros_like(Bsrc)
        Bv = torch.as_strided(B, (n, n), (1, n))
        c.register_input(Bv)
        C = torch.empty((n, rows), device=dev).t()
        ranks.append((A, Bv, C))
    torch.cuda.synchronize()

    def call():
        for r, c in enumerate(comms):
            A, Bv, C = ranks[r]
            emm.sgemm_multi(c, n, n, n, A, Bv, C, 1.0, 0.0, stream=streams[r])
        torch.cuda.synchronize()

    call()   # warm (workspaces)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        call()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    gemm = [(e.time_range.start, e.time_range.end) for e in ev if "tc_" in e.name and "kernel" in e.name]
    cpy = [(e.time_range.start, e.time_range.end) for e in ev if "Memcpy" in e.name and "DtoD" in e.name]
    t0 = min(s for s, _ in gemm + cpy)
    cbusy = sum(e - s for s, e in cpy)
    cover = sum(overlap(iv, gemm) for iv in cpy)
    out = {"P": P, "n": n, "gemm_kernels": len(gemm), "chunk_copies": len(cpy),
           "copy_busy_ms": cbusy / 1e3, "copy_time_under_gemm_ms": cover / 1e3,
           "copy_overlap_frac": cover / cbusy if cbusy else None,
           "first_gemm_ms": (min(s for s, _ in gemm) - t0) / 1e3,
           "span_ms": (max(e for _, e in gemm + cpy) - t0) / 1e3,
           "copy_GBps": (P - 1) * 4.0 * n * n / (cbusy * 1e-6) / 1e9 if cbusy else None}
    print(json.dumps(out))
    for c in comms:
        c.close()


if __name__ == "__main__":
    main()
