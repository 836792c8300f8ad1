#!/usr/bin/env python
"""Context numbers (NOT the product path, not a target): cuBLAS through
torch.matmul on the same B200 for square N^3, FP32 (precision 'highest': FP32
SGEMM) and TF32 ('high'), device time of one call with L2 flushed, median of
5, and their worst error vs the FP64 oracle relative to the 1e-5*S bound on a
few sampled rows (tests-style check; the oracle is test infrastructure)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))   # tests/ helper (uses the oracle)
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, device=dev)
    for n in (4096, 8192, 16384):
        A = datagen.matrix("uniform", datagen.TAG_A, n, n, device=dev)   # column-major views
        B = datagen.matrix("uniform", datagen.TAG_B, n, n, device=dev)
        rows = np.array([0, n // 2, n - 1])
        A_rows = datagen.storage_of(datagen.submatrix("uniform", datagen.TAG_A, n, n, rows)).numpy()
        Bh = datagen.storage_of(B).cpu().numpy()
        R, S, T, st = oracle.sgemm_sub("N", "N", len(rows), n, n, 1.0, A_rows, len(rows), Bh, n, 0.0, None, len(rows))
        for prec in ("highest", "high"):
            torch.set_float32_matmul_precision(prec)
            C = torch.matmul(A, B)
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                C = torch.matmul(A, B)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            G = C[rows].double().cpu().numpy()
            err = float(np.max(np.abs(G - R) / (1e-5 * S)))
            print(json.dumps({"n": n, "torch_precision": prec, "median_ms": ms,
                              "tflops": 2 * n ** 3 / ms / 1e9, "max_err_over_1e-5S": err}), flush=True)
        del A, B, C


if __name__ == "__main__":
    main()
