#!/usr/bin/env python3
"""Near-minimax polynomial fits for the encode kernel's FMA-pipe sin/cos (encode.cu
sincos_poly): sin(r) = r + r^3 P(r^2), cos(r) = 1 + r^2 Q(r^2) on [-pi/2, pi/2], by Lawson's
iteratively reweighted least squares; then checks the fp32 Horner evaluation error."""
import sys

import numpy as np

LITE = "--lite" in sys.argv   # the packed encode's cheaper pair: sin degree 7, cos degree 8

x = np.cos(np.linspace(0, np.pi, 4001)) * np.pi / 2
x = x[x >= 0]


def fit(f, powers, iters=200):
    A = np.stack([x ** p for p in powers], 1)
    w = np.ones_like(x)
    for _ in range(iters):
        c, *_ = np.linalg.lstsq(A * w[:, None], f * w, rcond=None)
        e = np.abs(A @ c - f)
        w = w * (e / e.max() + 1e-12) ** 0.5
        w /= w.max()
    return c


if LITE:
    cs = fit(np.sin(x) - x, [3, 5, 7])
    cc = fit(np.cos(x) - 1, [2, 4, 6, 8])
    f32 = np.float32
    r = np.linspace(-np.pi / 2, np.pi / 2, 200001).astype(f32)
    r2 = r * r
    S = [f32(v) for v in cs]
    C = [f32(v) for v in cc]
    p = S[2] * r2 + S[1]
    p = p * r2 + S[0]
    s = (p * r2) * r + r
    q = C[3] * r2 + C[2]
    q = q * r2 + C[1]
    q = q * r2 + C[0]
    c = q * r2 + f32(1)
    print("sin coefficients (r^3..r^7):", [f"{float(v):.9e}" for v in S])
    print("cos coefficients (r^2..r^8):", [f"{float(v):.9e}" for v in C])
    print("fp32 max error: sin %.3g cos %.3g" % (np.abs(s - np.sin(r.astype(np.float64))).max(),
                                               np.abs(c - np.cos(r.astype(np.float64))).max()))
    sys.exit(0)
cs = fit(np.sin(x) - x, [3, 5, 7, 9])
cc = fit(np.cos(x) - 1, [2, 4, 6, 8, 10])
f32 = np.float32
r = np.linspace(-np.pi / 2, np.pi / 2, 200001).astype(f32)
r2 = r * r
S = [f32(v) for v in cs]
C = [f32(v) for v in cc]
p = S[3] * r2 + S[2]
p = p * r2 + S[1]
p = p * r2 + S[0]
s = (p * r2) * r + r
q = C[4] * r2 + C[3]
q = q * r2 + C[2]
q = q * r2 + C[1]
q = q * r2 + C[0]
c = q * r2 + f32(1)
print("sin coefficients (r^3..r^9):", [f"{float(v):.9e}" for v in S])
print("cos coefficients (r^2..r^10):", [f"{float(v):.9e}" for v in C])
print("fp32 max error: sin %.3g cos %.3g" % (np.abs(s - np.sin(r.astype(np.float64))).max(),
                                           np.abs(c - np.cos(r.astype(np.float64))).max()))
