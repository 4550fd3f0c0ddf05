"""Vectorised numpy restatement of one ROW BAND of the 2D selective scan with
vertical carries at the band edges.  TEST INFRASTRUCTURE ONLY (the CPU compute
backend of the gloo row-band tests, never shipped or timed).

Same recurrences as the reference oracle:
  delta = softplus(z + bias)                         math.hpp:15-21, :76-79
  Abar  = exp(delta A),  u = (delta B) x             math.hpp:81-89
  hh(i,j) = Abar hh(i,j-1) + u                       reference.cpp:85-96
  h(i,j)  = Abar h(i-1,j) + hh(i,j)                  reference.cpp:98-107, h(-1,j) = h_top
  y = sum_d C h + D x                                reference.cpp:103-110
  G  = C dy + Abar(i+1,j) G(i+1,j)                   engine.cpp:321-323 (g_bottom below the band)
  Gh = G + Abar(i,j+1) Gh(i,j+1)                     engine.cpp:346-348
  dAbar = Gh hh(i,j-1) + G h(i-1,j), dA += dAbar delta Abar, ddelta, dB, dC, dx, dz,
  dbias, dD                                          engine.cpp:355-397
Shapes: x, z, dy [S,H,W]; B, C [S,H,W,N]; A [S,N]; D, bias [S]; carries [S,W,N].
"""
import numpy as np


def _disc(z, B, x, A, bias):
    v = z + bias[:, None, None]
    delta = np.where(v > 20.0, v, np.log1p(np.exp(np.minimum(v, 20.0))))
    a = np.exp(delta[..., None] * A[:, None, None, :])
    u = (delta[..., None] * B) * x[..., None]
    return v, delta, a, u


def _scans(a, u, h_top):
    S, H, W, N = a.shape
    hh = np.empty_like(u)
    run = np.zeros((S, H, N), u.dtype)
    for j in range(W):
        run = a[:, :, j] * run + u[:, :, j]
        hh[:, :, j] = run
    h = np.empty_like(u)
    run = np.zeros((S, W, N), u.dtype) if h_top is None else h_top.astype(u.dtype)
    for i in range(H):
        run = a[:, i] * run + hh[:, i]
        h[:, i] = run
    return hh, h


def band_forward(x, z, B, C, A, D, bias, h_top=None):
    _, _, a, u = _disc(z, B, x, A, bias)
    _, h = _scans(a, u, h_top)
    y = (C * h).sum(-1) + D[:, None, None] * x
    return y, h[:, -1].copy()


def band_backward(x, z, B, C, A, D, bias, h_top, dy, g_bottom=None):
    v, delta, a, u = _disc(z, B, x, A, bias)
    hh, h = _scans(a, u, h_top)
    S, H, W, N = a.shape
    G = np.empty_like(u)
    dn = np.zeros((S, W, N), u.dtype) if g_bottom is None else g_bottom.astype(u.dtype)
    for i in range(H - 1, -1, -1):
        G[:, i] = C[:, i] * dy[:, i, :, None] + dn
        dn = a[:, i] * G[:, i]
    g_top = dn
    Gh = np.empty_like(u)
    rho = np.zeros((S, H, N), u.dtype)
    for j in range(W - 1, -1, -1):
        Gh[:, :, j] = G[:, :, j] + rho
        rho = a[:, :, j] * Gh[:, :, j]
    h_up = np.concatenate([(np.zeros((S, 1, W, N)) if h_top is None else h_top[:, None]), h[:, :-1]], axis=1)
    hh_left = np.concatenate([np.zeros((S, H, 1, N)), hh[:, :, :-1]], axis=2)
    dab = Gh * hh_left + G * h_up
    dA = (dab * delta[..., None] * a).sum(axis=(1, 2))
    sgb = (Gh * B).sum(-1)
    ddelta = (dab * a * A[:, None, None, :]).sum(-1) + sgb * x
    dB = Gh * (delta * x)[..., None]
    dC = dy[..., None] * h
    dx = D[:, None, None] * dy + delta * sgb
    sig = 1.0 / (1.0 + np.exp(-v))
    dz = ddelta * sig
    return dx, dz, dA, dB, dC, (dy * x).sum(axis=(1, 2)), dz.sum(axis=(1, 2)), g_top
