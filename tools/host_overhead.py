#!/usr/bin/env python
"""Host-side enqueue cost of one emm call (GPU tool, not a test): the stream
is parked behind a long device sleep, then R calls are enqueued and timed on
the host (perf_counter); the GPU never stalls the host here, so the number
is the library's CPU cost per call (validation, planning, tensor-map
encodes, launch API).

    python tools/host_overhead.py [--reps 200]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402

SHAPES = [("c3-NN", 1531, 997, 2049, "N", "N", (13, 7, 5)), ("c3-TN", 1531, 997, 2049, "T", "N", (13, 7, 5)),
          ("1024", 1024, 1024, 1024, "N", "N", (0, 0, 0)), ("333", 333, 333, 333, "N", "N", (0, 0, 0)),
          ("64", 64, 64, 64, "N", "N", (0, 0, 0))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--maths", default="3xtf32,1xtf32,ffma")
    ap.add_argument("--ws", type=int, default=0, help="pass a caller workspace (no library scratch allocation)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    for name, M, N, K, tA, tB, pad in SHAPES:
        ra, ca = (M, K) if tA == "N" else (K, M)
        rb, cb = (K, N) if tB == "N" else (N, K)
        lda, ldb, ldc = ra + pad[0], rb + pad[1], M + pad[2]
        A = torch.rand(ca * lda, device=dev)
        B = torch.rand(cb * ldb, device=dev)
        C = torch.zeros(N * ldc, device=dev)
        L = emm.lib()
        for math in a.maths.split(","):
            fn = L.emm_sgemm_ex
            wsb = emm.workspace_bytes(tA, tB, M, N, K, math) if a.ws else 0
            ws = torch.empty(wsb // 4 + 512, device=dev) if wsb else None
            wsp = (ws.data_ptr() + (-ws.data_ptr()) % 1024) if wsb else None
            args = (tA.encode(), tB.encode(), M, N, K, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0,
                    C.data_ptr(), ldc, s.cuda_stream, emm.MATH[math], wsp, wsb)

            def call():
                return fn(*args)
            for _ in range(5):
                call()
            torch.cuda.synchronize()
            ts = []
            torch.cuda._sleep(int(2e9))   # ~1 s of device sleep
            for _ in range(a.reps):
                t0 = time.perf_counter()
                call()
                ts.append(time.perf_counter() - t0)
            torch.cuda.synchronize()
            n0 = emm.launch_count()
            call()
            torch.cuda.synchronize()
            print(f"{name:6s} {math:7s} host us/call: median {statistics.median(ts) * 1e6:7.2f}  "
                  f"min {min(ts) * 1e6:7.2f}  launches/call {emm.launch_count() - n0}", flush=True)
    # ctypes floor: a trivial exported call with the same marshalling path
    f = emm.lib().emm_launch_count
    ts = []
    for _ in range(1000):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    print(f"ctypes floor (emm_launch_count): median {statistics.median(ts) * 1e6:.2f} us")


if __name__ == "__main__":
    main()
