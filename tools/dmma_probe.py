"""Which evaluation order does the fp64 MMA (DMMA) implement?  Reads the
output of tools/dmma_probe (trials of A, B, C, D) and compares every D entry
with candidate formulas evaluated exactly (fractions.Fraction, then
round-to-nearest-even via float()):
  seq_fma   : fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))  (k ascending)
  rev_fma   : the same chain with k descending
  fused     : round(c + sum_k a_k b_k), one rounding
  dot_then_c: round(round(sum_k a_k b_k) + c)
Usage: ./dmma_probe N | python tools/dmma_probe.py"""
import struct
import sys
from fractions import Fraction as F

import numpy as np

raw = sys.stdin.buffer.read()
t = struct.unpack("i", raw[:4])[0]
arr = np.frombuffer(raw[4:], dtype=np.float64)
A = arr[:t * 32].reshape(t, 8, 4)
B = arr[t * 32:t * 64].reshape(t, 4, 8)
C = arr[t * 64:t * 128].reshape(t, 8, 8)
D = arr[t * 128:t * 192].reshape(t, 8, 8)


def fma(a, b, c):
    return float(F(a) * F(b) + F(c))


hits = {"seq_fma": 0, "rev_fma": 0, "fused": 0, "dot_then_c": 0}
total = 0
for q in range(t):
    for i in range(8):
        for j in range(8):
            a, b, c, d = A[q, i], B[q, :, j], C[q, i, j], D[q, i, j]
            total += 1
            x = c
            for kk in range(4):
                x = fma(a[kk], b[kk], x)
            hits["seq_fma"] += x == d
            x = c
            for kk in (3, 2, 1, 0):
                x = fma(a[kk], b[kk], x)
            hits["rev_fma"] += x == d
            ex = F(c) + sum(F(a[kk]) * F(b[kk]) for kk in range(4))
            hits["fused"] += float(ex) == d
            dot = float(sum(F(a[kk]) * F(b[kk]) for kk in range(4)))
            hits["dot_then_c"] += float(F(dot) + F(c)) == d
print({"entries": total, **{k: f"{v}/{total}" for k, v in hits.items()}})
