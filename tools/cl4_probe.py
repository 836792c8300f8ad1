#!/usr/bin/env python
"""Probe a GEMM configuration on one shape (GPU tool): integer-exact inputs,
bitwise check of sampled rows against the oracle; prints ok / mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from test_gpu_parity import Case  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402

M, N, K = map(int, sys.argv[1].split(","))
tA, tB = sys.argv[2], sys.argv[3]
case = Case(tA, tB, M, N, K, 1.0, 1.0, kind="ints", c_kind="ints")
rows = np.unique(np.r_[0:8, M // 2:M // 2 + 8, M - 8:M])
R, S, T, _ = case.oracle(rows=rows)
Cg = case.run(emm, "3xtf32")
G = case.logical(Cg)[rows]
ok = np.array_equal(G, R.astype(np.float32).astype(np.float64))
print(M, N, K, tA, tB, "ok" if ok else f"MISMATCH max {np.max(np.abs(G - R))}", flush=True)
