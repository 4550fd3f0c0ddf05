"""Randomised shape sweep (fixed seeds) of forward + backward against the fp64
oracle (-m gpu): catches planner / kernel-family edge cases -- odd widths,
partial tiles and strips, shared parameters (P < S) and shared B/C (G > 1),
N from 1 to 200, fp32 and fp64."""
import numpy as np
import pytest
import torch

from oracle_lib import Oracle, rel_error
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd


def _cases(n=60, seed=2412):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        N = int(rng.choice([1, 1, 2, 3, 4, 8, 16, 16, 32, 40, 150]))
        H = int(rng.integers(1, 40))
        W = int(rng.integers(1, 260 if N <= 16 else 60))
        G = int(rng.choice([1, 1, 2]))
        P_div = int(rng.choice([1, 1, 2]))  # P = S / P_div
        S = G * P_div * int(rng.integers(1, 3))
        dt = str(rng.choice(["f32", "f64"]))
        out.append((S, H, W, N, S // P_div, G, dt))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N,P,G,dtype", _cases())
def test_random_shapes(S, H, W, N, P, G, dtype):
    from paper_2412_00678_b200 import tiled_scan_2d_backward, tiled_scan_2d_forward

    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=4000 + H * 7 + W, dtype=dtype, P=P, G=G)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    res = tiled_scan_2d_forward(x, z, B, C, A, D, bias)
    g = tiled_scan_2d_backward(res.saved, dy)
    torch.cuda.synchronize()
    yg, gg = (1e-12, 1e-10) if dtype == "f64" else (1e-4, 1e-4)
    label = f"S={S} {H}x{W} N={N} P={P} G={G} {dtype}"
    assert rel_error(res.y.cpu().numpy(), oracle_fwd(orc, b, "f64")) <= yg, label
    ref = oracle_bwd(orc, b, "f64")
    got = dict(dx=g.dx, dz=g.dz_raw, dA=g.da, dB=g.db, dC=g.dc, dD=g.dd, dbias=g.dbias)
    for k, t in got.items():
        e = rel_error(t.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1))
        assert e <= gg, f"{label}: {k} rel {e:.3e}"


# Cases the long sweep (tools/stress_random.py) singled out, pinned with the
# strict gate: fp32 per-scan scalar sums (dbias, dD, dA) of the general warp
# kernels over many cells with shared parameters (round-1 outlier: N = 5,
# 28 x 226, P = 3 of S = 6, CarryState emission on -> warp forward kernel).
@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N,P,G,T,seed0,emit", [
    (6, 28, 226, 5, 3, 1, 16, 9000 + 31 * 6310, True),
    (6, 28, 226, 5, 3, 1, 16, 9000 + 31 * 6310, False),
    (4, 60, 400, 5, 2, 1, 5, 4242, True),
    (4, 60, 400, 100, 2, 1, 16, 4243, False),
    (3, 89, 419, 7, 1, 1, 16, 4244, True),
])
def test_sweep_outliers_strict(S, H, W, N, P, G, T, seed0, emit):
    from paper_2412_00678_b200 import tiled_scan_2d_backward, tiled_scan_2d_forward

    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=seed0, dtype="f32", P=P, G=G)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    res = tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=T, carries=emit)
    g = tiled_scan_2d_backward(res.saved, dy)
    torch.cuda.synchronize()
    assert rel_error(res.y.cpu().numpy(), oracle_fwd(orc, b, "f64")) <= 1e-4
    ref = oracle_bwd(orc, b, "f64")
    got = dict(dx=g.dx, dz=g.dz_raw, dA=g.da, dB=g.db, dC=g.dc, dD=g.dd, dbias=g.dbias)
    for k, t in got.items():
        e = rel_error(t.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1))
        assert e <= 1e-4, f"{k} rel {e:.3e}"
