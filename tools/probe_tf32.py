#!/usr/bin/env python
"""Probe (R7): what does tcgen05.mma kind::tf32 do with the low 13
mantissa bits of raw FP32 inputs?  Runs the 1xTF32 path with the pack pass
copying raw bits (EMM_DEBUG_RAW_BIG=1) on C = A*B with B = ones and single
distinguishing values in A, and reports truncate / round-nearest-even /
round-nearest-away.  Also reports the accumulation mode from a two-term sum.
"""
import os
import sys

os.environ["EMM_DEBUG_RAW_BIG"] = "1"
os.environ["EMM_SMALL_FLOPS"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402

u = 2.0 ** -10          # tf32 ulp at 1.0
cases = {
    "1+0.75ulp": 1 + 0.75 * u,      # trunc -> 1, RN -> 1+u, RNA -> 1+u
    "1+0.5ulp": 1 + 0.5 * u,        # trunc -> 1, RNE -> 1, RNA -> 1+u
    "1+1.5ulp": 1 + 1.5 * u,        # trunc -> 1+u, RNE -> 1+2u, RNA -> 1+2u
    "-(1+0.75ulp)": -(1 + 0.75 * u),
}
M, N, K = 256, 256, 32
res = {}
for name, val in cases.items():
    A = torch.zeros(K, M, device="cuda").t()      # column-major M x K
    A[:, 0] = val
    B = torch.zeros(N, K, device="cuda").t()      # K x N
    B[0, :] = 1.0
    C = torch.zeros(N, M, device="cuda").t()
    emm.sgemm(A, B, C, math="1xtf32")
    torch.cuda.synchronize()
    got = float(C[0, 0])
    mode = {1.0: "trunc", 1 + u: "RN(E/A)"}.get(abs(got), f"other({abs(got)!r})")
    if name == "1+0.5ulp":
        mode = {1.0: "trunc-or-RNE", 1 + u: "RNA"}.get(got, f"other({got!r})")
    if name == "1+1.5ulp":
        mode = {1 + u: "trunc", 1 + 2 * u: "RN(E/A)"}.get(got, f"other({got!r})")
    res[name] = (val, got, mode)
    print(f"{name:14s} in={val!r:22} out={got!r:22} -> {mode}")
print("verdict:", "TRUNCATE" if all("trunc" in r[2] for r in res.values()) else "ROUND" if all("RN" in r[2] for r in res.values()) else "MIXED")
