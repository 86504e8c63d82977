import torch, time
n=985527
dev='cuda'
a=torch.randn(n,dtype=torch.float64,device=dev); b=torch.randn_like(a); c=torch.randn_like(a); d=torch.randn_like(a)
big=torch.empty(64*1024*1024, dtype=torch.float64, device=dev)  # 512 MB flush
def t(f, reps=50, flush=True):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    tot=0
    for i in range(reps+3):
        if flush: big.fill_(i)
        s.record(); f(); e.record(); torch.cuda.synchronize()
        if i>=3: tot+=s.elapsed_time(e)
    return tot/reps*1000
for flush in (False, True):
    print('flush',flush)
    print(' copy a->b (15.8MB)', round(t(lambda: b.copy_(a), flush=flush),1),'us')
    print(' axpy b+=2a (23.7MB)', round(t(lambda: b.add_(a, alpha=2.0), flush=flush),1),'us')
    print(' zero (7.9MB)', round(t(lambda: b.zero_(), flush=flush),1),'us')
    x=torch.randn(8*n,dtype=torch.float64,device=dev); y=torch.empty_like(x)
    print(' copy 8x (126MB)', round(t(lambda: y.copy_(x), flush=flush),1),'us')
