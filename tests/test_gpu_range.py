"""Exponent range of the FP32-accurate paths (R19).

The split paths (3xTF32: big + small TF32 parts; TF32+BF16) keep the north_star
bound |C - R| <= 1e-5*S + 1e-6*T wherever the products and their split parts
stay FP32-normal, whatever the scale: inputs scaled by 1e-18 .. 1e17 (products
1e-36 .. 1e34) must pass exactly as unscaled ones.  Below that (products in
the subnormal range, < 1.2e-38) FP32 arithmetic itself cannot meet a bound
relative to S (`tools/range_probe.py` measurements in DESIGN.md R19), so no test
asserts there.  Every mode runs on the tensor-core / FFMA kernels
(EMM_SMALL_FLOPS=0), several tiles with ragged tails.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16", "ffma"])
@pytest.mark.parametrize("sa,sb", [(1e-18, 1e-18), (1e-9, 1e-9), (1e17, 1e17), (1e-30, 1e12), (1e20, 1e-25)])
def test_scaled_inputs_keep_the_bound(emm, monkeypatch, math, sa, sb):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    M, N, K = 700, 520, 600
    rng = np.random.default_rng(7)
    A = ((rng.random(M * K) * 2 - 1) * sa).astype(np.float32)
    B = ((rng.random(K * N) * 2 - 1) * sb).astype(np.float32)
    C = ((rng.random(M * N) * 2 - 1) * sa * sb).astype(np.float32)
    R, S, T, st = oracle.sgemm_sub("N", "N", M, N, K, 1.25, A, M, B, K, -0.5, C, M)
    assert st == 0
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    st = emm.sgemm_ptr("N", "N", M, N, K, 1.25, dA.data_ptr(), M, dB.data_ptr(), K, -0.5, dC.data_ptr(), M,
                       torch.cuda.current_stream().cuda_stream, math)
    torch.cuda.synchronize()
    assert st == 0
    G = dC.cpu().double().numpy().reshape(N, M).T
    bound = 1e-5 * S + 1e-6 * T
    err = np.abs(G - R)
    assert np.all(err <= bound), f"max err/bound {float(np.max(err / np.maximum(bound, 1e-300))):.3g}"
