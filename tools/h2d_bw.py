import torch, time
n = 2123366400 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device='cuda')
for chunks in (1, 8, 16, 32):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step = n // chunks
    for i in range(chunks):
        d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D {chunks} chunks: {ms:.2f} ms -> {n*4/ms/1e6:.1f} GB/s")
# two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t=time.time()
half = n//2
with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize(); dt=time.time()-t
print(f"H2D 2 streams: {dt*1e3:.2f} ms -> {n*4/dt/1e9:.1f} GB/s")
mh = torch.empty(530841600, dtype=torch.uint8).pin_memory(); md = torch.empty(530841600, dtype=torch.uint8, device='cuda')
torch.cuda.synchronize(); t=time.time(); mh.copy_(md, non_blocking=True); torch.cuda.synchronize(); dt=time.time()-t
print(f"D2H 0.53 GB: {dt*1e3:.2f} ms -> {530841600/dt/1e9:.1f} GB/s")
