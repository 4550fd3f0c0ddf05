"""Parity of every kernel family the planner can pick, forward and backward,
against the fp64 oracle (-m gpu):
  * tile kernels (scan2d_tile2.cuh): N in {4, 8, 16, 32}, fp32 (SH = 2) and
    fp64 (SH = 1); partial tiles (H not a multiple of the tile height),
    partial strips, one CTA per scan and several CTAs chained through global
    carries (> 13 strips);
  * N = 1 row-sweep kernels (scan2d_rows1.cuh): J in {4, 2, 1} columns per
    lane, 8/16/32-lane segments, odd widths that fall back to the warp
    kernels;
  * the plan actually taken is checked, so a silent fallback cannot pass.
"""
import numpy as np
import pytest
import torch

from oracle_lib import Oracle, rel_error
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd

F32_GATE = 1e-4
F64_Y_GATE = 1e-12
F64_G_GATE = 1e-10


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _run(orc, S, H, W, N, dtype, seed):
    from paper_2412_00678_b200.api import Scan2dOp

    b = make_batch(orc, S, H, W, N, seed0=seed, dtype=dtype)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    op = Scan2dOp(S, H, W, N, dtype=x.dtype, device="cuda")
    y = op.forward(x, z, B, C, A, D, bias).clone()
    grads = [t.clone() for t in op.backward(x, z, B, C, A, D, bias, dy)]
    torch.cuda.synchronize()
    return b, op, y, grads


def _check(orc, b, y, grads, dtype, label):
    yg, gg = (F64_Y_GATE, F64_G_GATE) if dtype == "f64" else (F32_GATE, F32_GATE)
    e = rel_error(y.cpu().numpy(), oracle_fwd(orc, b, "f64"))
    assert e <= yg, f"{label}: y rel {e:.3e}"
    ref = oracle_bwd(orc, b, "f64")
    for k, t in zip(("dx", "dz", "dA", "dB", "dC", "dD", "dbias"), grads):
        e = rel_error(t.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1))
        assert e <= gg, f"{label}: {k} rel {e:.3e}"


@pytest.mark.gpu
@pytest.mark.parametrize("N", [4, 8, 16, 32])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("H,W", [(37, 40), (9, 212), (5, 16), (14, 14), (7, 7), (23, 230)])
def test_tile_kernels(orc, N, dtype, H, W):
    """(W % 4 != 0: x / z / dy rows are not 16-byte aligned -> element copies)"""
    S = 3
    b, op, y, grads = _run(orc, S, H, W, N, dtype, seed=77 + N + H)
    plan = op.plan()
    assert plan["cols_per_chunk"] == 1 and plan["cols_per_warp"] == 16, plan  # tile kernels ran
    _check(orc, b, y, grads, dtype, f"tile N={N} {dtype} {H}x{W}")


@pytest.mark.gpu
@pytest.mark.parametrize("W", [4, 7, 12, 14, 28, 30, 56, 64, 100, 128, 33])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_rows1_kernels(orc, W, dtype):
    S, H = 9, 13
    b, op, y, grads = _run(orc, S, H, W, 1, dtype, seed=300 + W)
    plan = op.plan()
    if W == 33 or (dtype == "f64" and W > 64):  # no J puts the row on <= 32 lanes: warp kernels
        assert plan["spl_x100_plus_lpc"] != 0, plan
    else:
        assert plan["spl_x100_plus_lpc"] == 0 and plan["cols_per_warp"] == W, plan  # row-sweep kernels ran
    _check(orc, b, y, grads, dtype, f"rows1 W={W} {dtype}")


@pytest.mark.gpu
@pytest.mark.parametrize("N,W", [(33, 21), (48, 21), (64, 21), (100, 21), (128, 21), (64, 300), (128, 130)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_wide_state_warp_kernels(orc, N, W, dtype):
    """N in (32, 128]: the general warp kernels (up to 4 states x 32 lanes per chunk),
    single and chained column groups."""
    S, H = 2, 11
    b, op, y, grads = _run(orc, S, H, W, N, dtype, seed=500 + N)
    _check(orc, b, y, grads, dtype, f"warp N={N} {dtype}")


@pytest.mark.gpu
@pytest.mark.parametrize("N,W", [(129, 12), (200, 16), (256, 40), (300, 9), (2048, 4)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_state_groups_beyond_128(orc, N, W, dtype):
    """N > 128 (up to the reference's 2048): passes over state groups of <= 128."""
    S, H = 2, 7
    b, op, y, grads = _run(orc, S, H, W, N, dtype, seed=700 + N)
    _check(orc, b, y, grads, dtype, f"groups N={N} {dtype}")


@pytest.mark.gpu
def test_state_groups_shared_params():
    """N > 128 with per-channel parameters (P < S) and shared B/C (G > 1)."""
    from scan_cases import batch_to_torch as b2t

    o = Oracle()
    b = make_batch(o, 6, 6, 10, 150, seed0=9, dtype="f64", P=3, G=2)
    from paper_2412_00678_b200 import tiled_scan_2d_backward, tiled_scan_2d_forward

    (x, z, B, C, A, D, bias), dy = b2t(b, device="cuda")
    res = tiled_scan_2d_forward(x, z, B, C, A, D, bias)
    g = tiled_scan_2d_backward(res.saved, dy)
    torch.cuda.synchronize()
    assert rel_error(res.y.cpu().numpy(), oracle_fwd(o, b, "f64")) <= F64_Y_GATE
    ref = oracle_bwd(o, b, "f64")
    got = dict(dx=g.dx, dz=g.dz_raw, dA=g.da, dB=g.db, dC=g.dc, dD=g.dd, dbias=g.dbias)
    for k, t in got.items():
        assert rel_error(t.cpu().numpy().reshape(-1), np.asarray(ref[k]).reshape(-1)) <= F64_G_GATE, k


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N,P,dtype,T", [
    (6, 77, 20, 4, 3, "f32", 5),     # 4 scans per warp, last warp half empty
    (1, 24, 30, 4, 1, "f64", 64),    # 2 scans per warp, one empty segment
    (3, 45, 20, 260, 3, "f64", 16),  # state groups, the N = 4 remainder group
    (5, 19, 30, 8, 5, "f32", 7),
])
def test_emission_forward_then_backward(orc, S, H, W, N, P, dtype, T):
    """CarryState emission runs the warp forward (several scans per warp for
    narrow grids) and the residual it saves feeds the tile backward: segments
    past the last scan must not write the residual's boundary carries (found
    by tools/stress_random.py)."""
    from paper_2412_00678_b200 import tiled_scan_2d_backward, tiled_scan_2d_forward

    b = make_batch(orc, S, H, W, N, seed0=9000, dtype=dtype, P=P)
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    for _ in range(3):  # the failure was a race between segments: repeat
        res = tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=T, carries=True)
        g = tiled_scan_2d_backward(res.saved, dy)
        torch.cuda.synchronize()
        _check(orc, b, res.y, [g.dx, g.dz_raw, g.da, g.db, g.dc, g.dd, g.dbias], dtype,
               f"emit S={S} {H}x{W} N={N} {dtype} T={T}")


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N,label", [
    (37, 40, 200, 16, "one wave, balanced 4-warp runs: every scan straddles CTAs"),
    (31, 16, 1024, 16, "two waves of 13-warp CTAs -> one wave of 14-warp CTAs (last-wave fill)"),
    (150, 8, 56, 8, "one wave, runs over all SMs, 4-strip scans split across CTAs"),
])
def test_tile_launch_geometries(orc, S, H, W, N, label):
    """The launch geometries the planner picks by size (scan2d_kern.inc
    launch_tile): balanced one-wave launches whose scans straddle CTAs (their
    carries cross through the tagged global words, loaded a tile ahead) and
    multi-wave forwards widened to 14 warps -- forward and backward against
    the fp64 oracle."""
    b, op, y, grads = _run(orc, S, H, W, N, "f32", 5200 + S)
    _check(orc, b, y, grads, "f32", label)
