"""Debug helper: direct (in-place TMA) path vs oracle on integer inputs, per
trans combo and math mode; prints where results differ."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EMM_SMALL_FLOPS"] = "0"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402

M, N, K = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 256, 32))]
for force in ("0", "1"):
    os.environ["EMM_FORCE_PACK"] = force
    for math in ("1xtf32", "3xtf32", "tf32bf16"):
        for tA in "NT":
            for tB in "NT":
                ar, ac = (M, K) if tA == "N" else (K, M)
                br, bc = (K, N) if tB == "N" else (N, K)
                A = datagen.matrix("ints", 1, ar, ac)
                B = datagen.matrix("ints", 2, br, bc)
                R, S, T, _ = oracle.sgemm_sub(tA, tB, M, N, K, 1.0, A, ar, B, br, 0.0, None, M)
                dA = datagen.storage_of(A).cuda()
                dB = datagen.storage_of(B).cuda()
                dC = torch.zeros(M * N, device="cuda")
                st = emm.sgemm_ptr(tA, tB, M, N, K, 1.0, dA.data_ptr(), ar, dB.data_ptr(), br, 0.0, dC.data_ptr(), M,
                                   torch.cuda.current_stream().cuda_stream, math)
                torch.cuda.synchronize()
                G = dC.cpu().double().numpy().reshape(N, M).T
                bad = np.argwhere(G != R)
                msg = "ok" if len(bad) == 0 else f"{len(bad)} bad, first {bad[:3].tolist()} g={G[tuple(bad[0])]} r={R[tuple(bad[0])]}"
                rows = sorted(set(bad[:, 0].tolist()))[:8] if len(bad) else []
                cols = sorted(set(bad[:, 1].tolist()))[:8] if len(bad) else []
                print(f"force={force} {math:8s} {tA}{tB} st={st} {msg} rows={rows} cols={cols}", flush=True)
