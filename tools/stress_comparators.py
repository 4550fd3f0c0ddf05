"""Randomised sweep of the comparator operators (scan2d_forward_variant):
the naive 2D scan against the fp64 oracle, the flat 1D scan against a numpy
sequential scan of the row-major flattening (the reference's block_scan_1d
semantics, engine.cpp:489-526).

usage: python tools/stress_comparators.py <n_cases> [seed]"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from oracle_lib import Oracle, rel_error  # noqa: E402
from scan_cases import batch_to_torch, make_batch, oracle_fwd  # noqa: E402
import paper_2412_00678_b200._native as nat  # noqa: E402


def run_variant(b, variant, dtype):
    (x, z, B, Cc, A, D, bias), _ = batch_to_torch(b, dtype=dtype)
    desc = nat.make_desc(b.S, b.H, b.W, b.N, params_period=b.P, bc_group=b.G,
                         dtype=nat.F64 if dtype == torch.float64 else nat.F32)
    y = torch.empty_like(x)
    wsb = nat.lib.scan2d_comparator_workspace_bytes(C.byref(desc), variant)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    p = lambda t: C.c_void_p(t.data_ptr())
    rc = nat.lib.scan2d_forward_variant(C.byref(desc), variant, p(x), p(z), p(B), p(Cc), p(A), p(D), p(bias),
                                        p(y), p(ws), wsb, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != nat.OK:
        raise RuntimeError(f"status {rc}")
    torch.cuda.synchronize()
    return y.cpu().numpy()


def flat1d_ref(b):
    """h_t = Abar_t h_{t-1} + Bbar_t x_t over the row-major flattening, y = C.h + D x."""
    S, H, W, N = b.S, b.H, b.W, b.N
    y = np.empty((S, H, W))
    for s in range(S):
        p, g = s % b.P, s // b.G
        v = b.z[s].reshape(-1).astype(np.float64) + b.bias[p]
        d = np.where(v > 20, v, np.log1p(np.exp(np.minimum(v, 20))))
        Ab = np.exp(d[:, None] * b.A[p][None, :])
        u = (d[:, None] * b.B[g].reshape(-1, N)) * b.x[s].reshape(-1)[:, None]
        h = np.zeros(N)
        out = np.empty(H * W)
        Cf = b.C[g].reshape(-1, N)
        xf = b.x[s].reshape(-1)
        for t in range(H * W):
            h = Ab[t] * h + u[t]
            out[t] = Cf[t] @ h + b.D[p] * xf[t]
        y[s] = out.reshape(H, W)
    return y


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 9
    rng = np.random.default_rng(seed)
    orc = Oracle()
    fails, t0 = 0, time.time()
    for c in range(n):
        N = int(rng.choice([1, 2, 4, 5, 16, 32, 64]))
        H, W = int(rng.integers(1, 40)), int(rng.integers(1, 70))
        G = int(rng.choice([1, 1, 2]))
        S = G * int(rng.integers(1, 4))
        P = S
        dt = str(rng.choice(["f32", "f64"]))
        tdt = torch.float64 if dt == "f64" else torch.float32
        gate = 1e-12 if dt == "f64" else 1e-4
        label = f"#{c} S={S} {H}x{W} N={N} G={G} {dt}"
        try:
            b = make_batch(orc, S, H, W, N, seed0=300 + c, dtype=dt, P=P, G=G)
            e1 = rel_error(run_variant(b, nat.VARIANT_NAIVE, tdt), oracle_fwd(orc, b, "f64"))
            e2 = rel_error(run_variant(b, nat.VARIANT_FLAT1D, tdt), flat1d_ref(b))
            if e1 > gate or e2 > (gate if dt == "f32" else 1e-10):
                fails += 1
                print("FAIL", label, f"naive {e1:.2e} flat1d {e2:.2e}", flush=True)
        except Exception as exc:  # noqa: BLE001
            fails += 1
            print("ERROR", label, repr(exc)[:200], flush=True)
    print(f"comparators: {n} cases, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
