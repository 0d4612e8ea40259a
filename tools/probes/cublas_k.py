import torch
for n,k in [(16000,128),(16000,256),(8192,8192),(4096,96)]:
    a=torch.randn(n,k,dtype=torch.float64,device='cuda'); b=torch.randn(k,n,dtype=torch.float64,device='cuda')
    c=torch.empty(n,n,dtype=torch.float64,device='cuda')
    for _ in range(3): torch.matmul(a,b,out=c)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): torch.matmul(a,b,out=c)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/5
    print(n,k, f"{ms:.3f} ms", f"{2*n*n*k/ms/1e9:.1f} TF/s")
