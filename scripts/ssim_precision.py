"""Precision of the loss kernels' arithmetic, emulated in numpy on the golden
loss cases (CPU): the SSIM image gradient with (a) float64 moments and fp32
unshifted seeds (the round-1 kernels) and (b) fp32 moments of values shifted
by 0.5 with seeds in the shifted variables (the current ssim_stats), both
with float64 adjoint filtering (ssim_grad), against the float64 oracle.
Prints the largest elementwise relative deviation over the gradient entries
above 1e-3 of the largest."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cgs_oracle as O  # noqa: E402

k64 = np.exp(-0.5 * ((np.arange(11) - 5) / 1.5) ** 2)
k64 /= k64.sum()
k32 = k64.astype(np.float32)
C1, C2 = 1e-4, 9e-4


def filt(x, k):  # valid separable filter, horizontal pass first (the kernels' order)
    H, W = x.shape
    rows = sum(k[j] * x[:, j:W - 10 + j] for j in range(11))
    return sum(k[j] * rows[j:H - 10 + j, :] for j in range(11))


def adj(g, shape):  # adjoint, float64
    pad = np.zeros((shape[0] + 10, shape[1] + 10))
    pad[10:-10, 10:-10] = g
    return filt(pad, k64)


def grad_round1(a, b):
    g, n = np.zeros_like(a), 0
    for c in range(a.shape[2]):
        x, y = a[:, :, c], b[:, :, c]
        mx, my, A1, A2, B1, B2 = O._ssim_terms(x, y)
        F = 1.0 / (B1 * B2)
        s = A1 * A2 * F
        f32 = lambda t: t.astype(np.float32).astype(np.float64)  # noqa: E731
        d_mx = f32(2 * my * F * (A2 - A1) - 2 * mx * s * (1.0 / B1 - 1.0 / B2))
        d_ex2, d_exy = f32(-s / B2), f32(2 * A1 * F)
        g[:, :, c] = adj(d_mx, x.shape) + 2 * x * adj(d_ex2, x.shape) + y * adj(d_exy, x.shape)
        n += s.size
    return g / n


def grad_shifted32(a, b):
    g, n = np.zeros_like(a), 0
    for c in range(a.shape[2]):
        x, y = a[:, :, c] - 0.5, b[:, :, c] - 0.5
        xf, yf = x.astype(np.float32), y.astype(np.float32)
        m0, m1, m2, m3, m4 = [filt(t, k32).astype(np.float64) for t in (xf, yf, xf * xf, yf * yf, xf * yf)]
        vx, vy, cxy = m2 - m0 * m0, m3 - m1 * m1, m4 - m0 * m1
        mx, my = m0 + 0.5, m1 + 0.5
        A1, A2 = 2 * mx * my + C1, 2 * cxy + C2
        B1, B2 = mx * mx + my * my + C1, vx + vy + C2
        F = 1.0 / (B1 * B2)
        s = A1 * A2 * F
        d_var, d_cov = -s / B2, 2 * A1 * F
        d0 = s * (2 * my / A1 - 2 * mx / B1) - 2 * m0 * d_var - m1 * d_cov
        f32 = lambda t: t.astype(np.float32).astype(np.float64)  # noqa: E731
        g[:, :, c] = adj(f32(d0), x.shape) + 2 * x * adj(f32(d_var), x.shape) + y * adj(f32(d_cov), x.shape)
        n += s.size
    return g / n


d = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                         "golden", "loss_sh.npz"))
for name, fn in (("round 1: fp64 moments, fp32 seeds", grad_round1),
                 ("now: fp32 shifted moments, fp32 shifted seeds", grad_shifted32)):
    worst = 0.0
    for kk in range(4):
        a, b = d[f"loss{kk}_a"].astype(np.float64), d[f"loss{kk}_b"].astype(np.float64)
        if a.ndim == 2:
            a, b = a[:, :, None], b[:, :, None]
        ref, got = O.ssim_grad(a, b), fn(a, b)
        big = np.abs(ref) > 1e-3 * np.abs(ref).max()
        worst = max(worst, float((np.abs(got - ref)[big] / np.abs(ref)[big]).max()))
    print(f"{name:48s} max rel deviation {worst:.2e}")
