import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(7)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    part = n // streams
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for k, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[k*part:(k+1)*part].copy_(h[k*part:(k+1)*part], non_blocking=True)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"H2D {streams} stream(s): {n/t/1e9:.1f} GB/s")
torch.cuda.synchronize(); t0=time.perf_counter(); h.copy_(d); torch.cuda.synchronize(); print(f"D2H: {n/(time.perf_counter()-t0)/1e9:.1f} GB/s")
