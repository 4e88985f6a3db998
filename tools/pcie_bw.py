"""Pinned H2D / D2H bandwidth on this box: alone, concurrent, and in chunks."""
import json

import torch

N = 2 * 10**9 // 4
h = torch.empty(N, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(N, dtype=torch.float32, pin_memory=True)
d = torch.empty(N, dtype=torch.float32, device="cuda")
d2 = torch.empty(N, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {}
out["h2d_GBs"] = 8.0 / timed(lambda: d.copy_(h, non_blocking=True))  # 2 GB / ms -> GB/s*1e-3
out["h2d_GBs"] = 2e9 / (timed(lambda: d.copy_(h, non_blocking=True)) / 1e3) / 1e9
out["d2h_GBs"] = 2e9 / (timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e3) / 1e9


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


out["concurrent_each_GBs"] = 2e9 / (timed(both) / 1e3) / 1e9
CH = 8 * 10**6  # 32 MB chunks


def chunked():
    for c in range(0, N, CH):
        h2[c:c + CH].copy_(d2[c:c + CH], non_blocking=True)


out["d2h_32MB_chunks_GBs"] = 2e9 / (timed(chunked) / 1e3) / 1e9
print(json.dumps(out))
