import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import make_w_device
n, m, k = 1_000_000, 500, 1500
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
W = make_w_device(n, m, 1e-10, 0, torch.float32, "cuda")
st = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0)
st.factorize_columns(W, W.shape[1], m)
torch.cuda.synchronize()
st.m = 0
t0 = time.perf_counter(); st._enqueue_factorization(W, W.shape[1], m); t1 = time.perf_counter()
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0):.1f} ms ({1e6*(t1-t0)/m:.1f} us/column), total {1e3*(t2-t0):.1f} ms")
