import torch, time, json
n = 2 * 1024**3 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda"); d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); out["h2d_GBps"] = 8.0 / 4 * 2**30 * 4 / (time.perf_counter() - t) / 1e9 if False else (n * 4) / (time.perf_counter() - t) / 1e9
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); out["d2h_GBps"] = (n * 4) / (time.perf_counter() - t) / 1e9
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); out["both_each_GBps"] = (n * 4) / (time.perf_counter() - t) / 1e9
    # chunked 4 MB H2D copies (the e2e pattern)
    torch.cuda.synchronize(); t = time.perf_counter()
    c = 1024 * 1024
    with torch.cuda.stream(s1):
        for o in range(0, n, c): d[o:o + c].copy_(h[o:o + c], non_blocking=True)
    torch.cuda.synchronize(); out["h2d_4MB_chunks_GBps"] = (n * 4) / (time.perf_counter() - t) / 1e9
print(json.dumps(out))
