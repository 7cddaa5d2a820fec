import torch
n=64<<20
h=[torch.empty(n,dtype=torch.uint8,pin_memory=True) for _ in range(2)]
d=[torch.empty(n,dtype=torch.uint8,device='cuda') for _ in range(2)]
ss=[torch.cuda.Stream() for _ in range(2)]
for k in (1,2):
    for _ in range(3):
        torch.cuda.synchronize()
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record()
        for j in range(k):
            ss[j].wait_event(a)
            with torch.cuda.stream(ss[j]):
                for r in range(10): d[j].copy_(h[j],non_blocking=True)
        for j in range(k): torch.cuda.current_stream().wait_stream(ss[j])
        b.record(); torch.cuda.synchronize()
    print('streams',k,'GB/s',k*10*n/(a.elapsed_time(b)/1e3)/1e9)
