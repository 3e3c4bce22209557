import torch, time
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device='cuda'); h = torch.empty(n, dtype=torch.uint8).pin_memory()
for it in range(3):
    torch.cuda.synchronize(); t = time.time(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt = time.time() - t
    print(f"D2H 1 GiB: {n/dt/1e9:.1f} GB/s")
    torch.cuda.synchronize(); t = time.time(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt = time.time() - t
    print(f"H2D 1 GiB: {n/dt/1e9:.1f} GB/s")
# 32 chunks of 32 MiB on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.time()
for i in range(32):
    with torch.cuda.stream(s1 if i % 2 else s2):
        h[i << 25:(i + 1) << 25].copy_(d[i << 25:(i + 1) << 25], non_blocking=True)
torch.cuda.synchronize(); dt = time.time() - t
print(f"D2H 32 x 32 MiB two streams: {n/dt/1e9:.1f} GB/s")
