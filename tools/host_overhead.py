import time, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1912_04379_b200 as emm
for n in (64, 512, 1024):
    A = torch.rand(n, n, device="cuda").t(); B = torch.rand(n, n, device="cuda").t(); C = torch.empty(n, n, device="cuda").t()
    ws = torch.empty(max(emm.workspace_bytes("N","N",n,n,n,"3xtf32"),1)+1024, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    L = emm.lib()
    args = (b"N", b"N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, s, 0, (ws.data_ptr()+1023)//1024*1024, ws.numel()-1024)
    for _ in range(50): L.emm_sgemm_ex(*args)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); N = 2000
    for _ in range(N): L.emm_sgemm_ex(*args)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"n={n}: host enqueue {1e6*(t1-t0)/N:.2f} us/call, wall incl. GPU {1e6*(t2-t0)/N:.2f} us/call")
