"""Shared fixtures for the parity tests: batched instances built from the
reference generator (random_instance, fixtures.hpp:20-37, restated in
oracle/scan2d_oracle.c) and helpers to run the GPU path and the oracle on the
same inputs.  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle_lib import Oracle


@dataclass
class Batch:
    S: int
    H: int
    W: int
    N: int
    P: int
    G: int
    x: np.ndarray  # [S,H,W]
    z: np.ndarray
    B: np.ndarray  # [S/G,H,W,N]
    C: np.ndarray
    A: np.ndarray  # [P,N]
    D: np.ndarray  # [P]
    bias: np.ndarray
    dy: np.ndarray  # [S,H,W]


def make_batch(orc: Oracle, S, H, W, N, seed0=1000, dtype="f64", P=None, G=1) -> Batch:
    """Scan s uses random_instance(H, W, N, seed0 + s); params come from scan
    p's instance (p < P), B/C from scan g*G's instance; dy from
    Rng(seed ^ 0x5eed) as in gradcheck.cpp:53-55."""
    P = S if P is None else P
    dt = np.float64 if dtype == "f64" else np.float32
    x = np.empty((S, H, W), dt)
    z = np.empty((S, H, W), dt)
    B = np.empty((S // G, H, W, N), dt)
    C = np.empty((S // G, H, W, N), dt)
    A = np.empty((P, N), dt)
    D = np.empty((P,), dt)
    bias = np.empty((P,), dt)
    dy = np.empty((S, H, W), dt)
    for s in range(S):
        inst = orc.random_instance(H, W, N, seed0 + s, dtype)
        x[s] = inst.x.reshape(H, W)
        z[s] = inst.z.reshape(H, W)
        if s % G == 0:
            B[s // G] = inst.B.reshape(H, W, N)
            C[s // G] = inst.C.reshape(H, W, N)
        if s < P:
            A[s] = inst.A
            D[s] = inst.D
            bias[s] = inst.bias
        dy[s] = orc.fill_normal((seed0 + s) ^ 0x5EED, H * W, dtype).reshape(H, W)
    return Batch(S, H, W, N, P, G, x, z, B, C, A, D, bias, dy)


def batch_to_torch(b: Batch, device="cuda", dtype=None):
    import torch

    tdt = dtype or (torch.float64 if b.x.dtype == np.float64 else torch.float32)
    conv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=tdt)
    return [conv(v) for v in (b.x, b.z, b.B, b.C, b.A, b.D, b.bias)], conv(b.dy)


def oracle_fwd(orc: Oracle, b: Batch, dtype="f64", threads=8):
    cast = (lambda a: a.astype(np.float64)) if dtype == "f64" else (lambda a: a.astype(np.float32))
    y = orc.fwd_batch(b.S, b.P, b.G, b.H, b.W, b.N, *[cast(v) for v in (b.x, b.z, b.B, b.C, b.A, b.D, b.bias)],
                      dtype=dtype, threads=threads)
    return y.reshape(b.S, b.H, b.W)


def oracle_bwd(orc: Oracle, b: Batch, dtype="f64"):
    cast = (lambda a: a.astype(np.float64)) if dtype == "f64" else (lambda a: a.astype(np.float32))
    out = orc.bwd_batch(b.S, b.P, b.G, b.H, b.W, b.N,
                        *[cast(v) for v in (b.x, b.z, b.B, b.C, b.A, b.D, b.bias, b.dy)], dtype=dtype)
    return out
