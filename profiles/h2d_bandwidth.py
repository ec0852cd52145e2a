import torch, time
torch.cuda.init()
n = 288 * 1024 * 1024 // 8
hs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(3)]
ds = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
ss = [torch.cuda.Stream() for _ in range(3)]
for k in (1, 2, 3):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i in range(3):
            s = ss[i % k]
            with torch.cuda.stream(s):
                ds[i].copy_(hs[i], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{k} stream(s): 3 x 288MB in {dt*1e3:.1f} ms = {3*288/1024/dt:.1f} GB/s")
# chunked on one stream
torch.cuda.synchronize(); t = time.perf_counter()
for i in range(3):
    for c in range(8):
        ds[i][c*n//8:(c+1)*n//8].copy_(hs[i][c*n//8:(c+1)*n//8], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"chunked: {3*288/1024/dt:.1f} GB/s")
