import torch, time, json, sys
sys.path.insert(0,'/root/repo')
out={}
for mb in (64, 256, 1024, 4096):
    h=torch.empty(mb<<20,dtype=torch.uint8).pin_memory(); d=torch.empty(mb<<20,dtype=torch.uint8,device='cuda')
    for _ in range(2): d.copy_(h,non_blocking=True)
    torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(5): d.copy_(h,non_blocking=True)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/5
    out[f'h2d_pinned_{mb}MB_gbs']=round((mb<<20)/dt/1e9,2)
    del h,d
# two streams concurrently
h1=torch.empty(1<<30,dtype=torch.uint8).pin_memory(); h2=torch.empty(1<<30,dtype=torch.uint8).pin_memory()
d1=torch.empty(1<<30,dtype=torch.uint8,device='cuda'); d2=torch.empty(1<<30,dtype=torch.uint8,device='cuda')
s1,s2=torch.cuda.Stream(),torch.cuda.Stream()
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1): d1.copy_(h1,non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2,non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/3
out['h2d_two_streams_gbs']=round((2<<30)/dt/1e9,2)
print(json.dumps(out))
