import torch, time
n = 154140672
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]
for k in (1, 2, 4):
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for it in range(10):
            ch = n // k
            for j in range(k):
                with torch.cuda.stream(s[j]):
                    d[j*ch:(j+1)*ch].copy_(h[j*ch:(j+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 10
    print(f"{k} streams: {n / t / 1e9:.1f} GB/s")
