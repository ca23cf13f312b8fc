import torch, time
def t(f, n=5):
    f(); torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(n):
        s.record(); f(); e.record(); torch.cuda.synchronize(); best=min(best, s.elapsed_time(e))
    return best
N=8192
a=torch.randn(N,N,dtype=torch.float64,device='cuda'); b=torch.randn(N,N,dtype=torch.float64,device='cuda')
ms=t(lambda: a@b); print(f"cuBLAS DGEMM {N}^3: {2*N**3/ms/1e9:.2f} TF")
for n,B in [(1600,148),(400,2304),(100,256*8)]:
    A=torch.randn(B,n,n,dtype=torch.float64,device='cuda')+n*torch.eye(n,dtype=torch.float64,device='cuda')
    ms=t(lambda: torch.linalg.lu_factor(A), 3); print(f"torch batched lu_factor n={n} B={B}: {ms:.2f} ms  {B*2/3*n**3/ms/1e9:.2f} TF")
