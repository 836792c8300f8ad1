#!/usr/bin/env python
"""GPU tool (not a test): max error / (1e-5 S) of every math mode vs the oracle when A and B are
scaled toward the FP32 subnormal range (512^3, EMM_SMALL_FLOPS=0).  DESIGN.md R19."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1912_04379_b200 as emm, oracle
M = N = K = 512
os.environ["EMM_SMALL_FLOPS"] = "0"
rng = np.random.default_rng(0)
for scale in [1e-17, 1e-18, 1e-19, 1e-20, 1e-21, 1e-22, 1e-23]:
    A = (rng.random(M * K, dtype=np.float32) * scale).astype(np.float32)
    B = (rng.random(K * N, dtype=np.float32) * scale).astype(np.float32)
    R, S, T, st = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, None, M)
    out = []
    for math in ["3xtf32", "tf32bf16", "ffma", "1xtf32"]:
        dA = torch.from_numpy(A).cuda(); dB = torch.from_numpy(B).cuda(); dC = torch.zeros(M * N, device="cuda")
        st = emm.sgemm_ptr("N", "N", M, N, K, 1.0, dA.data_ptr(), M, dB.data_ptr(), K, 0.0, dC.data_ptr(), M,
                           torch.cuda.current_stream().cuda_stream, math)
        torch.cuda.synchronize()
        G = dC.cpu().double().numpy().reshape(N, M).T
        err = np.abs(G - R); bound = 1e-5 * S
        out.append(f"{math}:{float(np.max(err / np.maximum(bound, 1e-300))):.3g}")
    print(f"A, B scale {scale:g}: max err / (1e-5 S):", " ".join(out), flush=True)
