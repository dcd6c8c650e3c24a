import torch, time
def t(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/n
M=307200
for K,N in ((105,64),(112,64),(64,357),(64,360)):
    x=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); w=torch.randn(N,K,device='cuda',dtype=torch.bfloat16)
    g=torch.randn(M,N,device='cuda',dtype=torch.bfloat16)
    fwd=t(lambda: x@w.t()); dx=t(lambda: g@w); dw=t(lambda: g.t()@x)
    print(f"K={K} N={N}: fwd {fwd:.3f} ms  dX {dx:.3f} ms  dW {dw:.3f} ms")
