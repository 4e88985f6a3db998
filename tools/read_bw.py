"""Pure-read HBM bandwidth on this B200 (torch reductions over 8 GiB) next to
the driver's copy figure, to bound what a read-dominated stream can reach."""
import torch
x = torch.empty(2 << 30, dtype=torch.float32, device="cuda").uniform_()
y = torch.empty_like(x)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best
nbytes = x.numel() * 4
print("sum (read)  GB/s", nbytes / (t(lambda: x.sum()) / 1e3) / 1e9)
print("copy (r+w)  GB/s", 2 * nbytes / (t(lambda: y.copy_(x)) / 1e3) / 1e9)
print("amax (read) GB/s", nbytes / (t(lambda: x.abs().max() if False else torch.amax(x)) / 1e3) / 1e9)
