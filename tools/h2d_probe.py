import torch, time, json
torch.cuda.set_device(0)
N = 1 << 30  # 1 GiB
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
res = {}
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = 64 << 20
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, off in enumerate(range(0, N, chunk)):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    res[f"streams_{ns}"] = round(N / el / 1e9, 2)
for chunk_mb in (8, 32, 128, 512):
    chunk = chunk_mb << 20
    s = torch.cuda.Stream()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for off in range(0, N, chunk):
            d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
    torch.cuda.synchronize(); el = time.perf_counter() - t0
    res[f"chunk_{chunk_mb}MB"] = round(N / el / 1e9, 2)
print(json.dumps(res))
