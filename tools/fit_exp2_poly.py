"""Fit the degree-3 polynomial used by the kernel's FMA-pipe exp2 (Exp2Poly).

2^f ~= 1 + f*(c1 + f*(c2 + f*c3)) on f in [-0.5, 0.5] (round-to-nearest range
reduction), constrained p(0) = 1, near-minimax in relative error via iteratively
re-weighted least squares. Prints the fp32 coefficients and the max relative error
evaluated in fp32 (1.0e-4).
"""
import numpy as np

f = np.linspace(-0.5, 0.5, 20001)
t = 2.0 ** f
A = np.stack([f, f ** 2, f ** 3], 1) / t[:, None]
b = (t - 1) / t
w = np.ones_like(f)
for _ in range(200):
    W = np.sqrt(w)
    c, *_ = np.linalg.lstsq(A * W[:, None], b * W, rcond=None)
    e = np.abs(A @ c - b)
    w = w * (e / e.max() + 1e-3) ** 0.5
    w /= w.mean()
c = c.astype(np.float32)
f32 = f.astype(np.float32)
p32 = np.float32(1) + f32 * (c[0] + f32 * (c[1] + f32 * c[2]))
print("c1, c2, c3 =", [float(x) for x in c])
print("max relative error (fp32 evaluation):", float(np.abs(p32.astype(np.float64) / t - 1).max()))
