import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_1912_04379_b200 as emm
M=N=K=64
A=torch.randn(M*K,device='cuda'); B=torch.randn(K*N,device='cuda'); C=torch.zeros(M*N,device='cuda')
cs=torch.cuda.Stream()
g=torch.cuda.CUDAGraph()
with torch.cuda.stream(cs):
    print("pre", emm.sgemm_ptr("N","N",M,N,K,1.0,A.data_ptr(),M,B.data_ptr(),K,0.0,C.data_ptr(),M,cs.cuda_stream,"3xtf32"))
    cs.synchronize()
    sts=[]
    with torch.cuda.graph(g, stream=cs):
        for _ in range(3):
            sts.append(emm.sgemm_ptr("N","N",M,N,K,1.0,A.data_ptr(),M,B.data_ptr(),K,0.0,C.data_ptr(),M,cs.cuda_stream,"3xtf32"))
print("in-capture statuses", sts, [emm.strerror(s) for s in sts])
C.zero_(); torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
print("after replay nonzero:", int((C!=0).sum()))
