import torch, time
n=1024*1000*1000//4
h=torch.empty(n,dtype=torch.float32).pin_memory(); h.fill_(1.0)
d=torch.empty(n,dtype=torch.float32,device='cuda')
for i in range(5):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h,non_blocking=True); e.record(); torch.cuda.synchronize()
    print('pinned H2D 1.024GB ms', s.elapsed_time(e), 'GB/s', 1.024/(s.elapsed_time(e)/1e3))
