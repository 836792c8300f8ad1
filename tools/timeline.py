#!/usr/bin/env python
"""Per-CTA timeline of one tc_sgemm_kernel launch (debug build only).

    EMM_TIMELINE=1 python -m paper_1912_04379_b200.build
    EMM_LIB=libemm_tl.so python tools/timeline.py --shape 1024,1024,1024,N,N

Slots (%globaltimer ns, relative to the earliest CTA entry):
  0 entry   1 prologue done (TMEM alloc, barriers, cluster sync)
  2 after griddepcontrol.wait   3 MMA: first stage ready (leader CTAs)
  4 MMA: last commit issued (leader CTAs)   5 epilogue: first accumulator ready
  6 epilogue: stores done   7 exit (after the final cluster sync)
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("EMM_LIB", "libemm_tl.so")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402

NAMES = ["entry", "prologue", "gdc_wait", "mma_first", "mma_last", "epi_first", "epi_done", "exit",
         "mbar_init", "tmem_alloc", "cluster_sync", "-"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1024,1024,1024,N,N")
    ap.add_argument("--math", default="3xtf32")
    ap.add_argument("--flush", type=int, default=1)
    ap.add_argument("--xs", type=int, default=1, help="read the KN1X (k_tcx.cu) timeline, else KN1's")
    a = ap.parse_args()
    M, N, K, tA, tB = a.shape.split(",")
    M, N, K = int(M), int(N), int(K)
    dev = torch.device("cuda", 0)
    L = emm.lib()
    tl = L.emm_debug_timeline_xs if a.xs else L.emm_debug_timeline
    tl.argtypes = [ctypes.c_void_p, ctypes.c_int]
    tl.restype = ctypes.c_int
    ra, ca = (M, K) if tA == "N" else (K, M)
    rb, cb = (K, N) if tB == "N" else (N, K)
    A = torch.rand(ca, ra, device=dev).t()
    B = torch.rand(cb, rb, device=dev).t()
    C = torch.zeros(N, M, device=dev).t()
    ws = torch.empty(emm.workspace_bytes(tA, tB, M, N, K, a.math), dtype=torch.uint8, device=dev)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, device=dev)
    for rep in range(4):
        if a.flush:
            flush.fill_(1.0)
        torch.cuda.synchronize()
        buf = np.zeros(512 * 12, dtype=np.uint64)
        tl(buf.ctypes.data, 0)
        emm.sgemm_ex(A, B, C, 1.0, 0.0, tA, tB, math=a.math, workspace=ws)
        torch.cuda.synchronize()
        st = tl(buf.ctypes.data, buf.size)
        assert st == 0
    t = buf.reshape(512, 12).astype(np.int64)
    ncta = int(np.count_nonzero(t[:, 0]))
    t = t[:ncta]
    t0 = t[:, 0].min()
    print(f"shape {M}x{N}x{K} {tA}{tB} {a.math}: {ncta} CTAs (last rep)")
    for s, nm in enumerate(NAMES):
        v = t[:, s]
        v = v[v > 0] - t0
        if v.size:
            print(f"  {s} {nm:10s} min {v.min() / 1e3:8.2f} us  median {np.median(v) / 1e3:8.2f}  max {v.max() / 1e3:8.2f}")


if __name__ == "__main__":
    main()
