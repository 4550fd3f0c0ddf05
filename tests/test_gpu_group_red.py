"""Shared-B/C backward with in-place group reductions (desc flag
SCAN2D_FLAG_GROUP_RED, -m gpu): dB / dC summed over each B/C group by L2
reductions from inside the tile backward instead of per-scan gradients plus
the fixed-order reduction kernel (model layout, SURVEY.md §8 f2,
model.cpp:174-193).  Against the fp64 oracle at the usual gates, and against
the deterministic path: the per-scan outputs (dx, dz, dA, dD, dbias) are the
same bits, dB / dC agree to summation-order rounding."""
import numpy as np
import pytest
import torch

from oracle_lib import Oracle, rel_error
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd

NAMES = ("dx", "dz", "dA", "dB", "dC", "dD", "dbias")
# (S, H, W, N, P, G, dtype): tile shapes (N in 4/8/16/32, several strips, ragged
# widths), a P < S case, fp64, and N = 5 / N = 1 where the flag is ignored
CASES = [(8, 40, 56, 16, 8, 8, "f32"), (12, 24, 200, 16, 12, 4, "f32"), (6, 33, 47, 8, 3, 3, "f32"),
         (4, 16, 16, 4, 4, 2, "f32"), (4, 20, 40, 32, 4, 4, "f32"), (6, 24, 40, 16, 6, 6, "f64"),
         (4, 10, 12, 5, 4, 2, "f32"), (8, 14, 14, 1, 8, 4, "f32")]


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def _run(b, dt, group_red):
    from paper_2412_00678_b200.api import Scan2dOp

    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, device="cuda")
    op = Scan2dOp(b.S, b.H, b.W, b.N, params_period=b.P, bc_group=b.G, dtype=dt, device="cuda",
                  group_red=group_red)
    y = op.forward(x, z, B, C, A, D, bias).cpu().numpy()
    g = dict(zip(NAMES, [t.cpu().numpy() for t in op.backward(x, z, B, C, A, D, bias, dy)]))
    # a second backward into the same buffers: the in-place sums start from zero every call
    g2 = dict(zip(NAMES, [t.cpu().numpy() for t in op.backward(x, z, B, C, A, D, bias, dy)]))
    return y, g, g2


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_group_red_vs_oracle_and_deterministic_path(orc, case):
    S, H, W, N, P, G, dts = case
    dt = torch.float64 if dts == "f64" else torch.float32
    b = make_batch(orc, S, H, W, N, seed0=4100, dtype=dts, P=P, G=G)
    y0, g0, _ = _run(b, dt, False)
    y1, g1, g1b = _run(b, dt, True)
    np.testing.assert_array_equal(y0, y1)
    for k in ("dx", "dz", "dA", "dD", "dbias"):
        np.testing.assert_array_equal(g0[k], g1[k], err_msg=k)
    tol_sum = 1e-12 if dts == "f64" else 2e-6
    for k in ("dB", "dC"):
        assert rel_error(g1[k].reshape(-1), g0[k].reshape(-1)) <= tol_sum, k
        assert rel_error(g1b[k].reshape(-1), g1[k].reshape(-1)) <= tol_sum, k
    gate = 1e-12 if dts == "f64" else 1e-4
    assert rel_error(y1.reshape(-1), oracle_fwd(orc, b, "f64").reshape(-1)) <= gate
    ref = oracle_bwd(orc, b, "f64")
    for k in NAMES:
        assert rel_error(g1[k].reshape(-1), np.asarray(ref[k]).reshape(-1)) <= gate, k


@pytest.mark.gpu
def test_group_red_model_layout_full_size(orc):
    """cfg2m's shape (one slide, D = 128 channels sharing B / C, 200 x 200,
    N = 16), gradients against the deterministic path and the fp64 oracle on
    the group sums."""
    S, H, W, N = 128, 200, 200, 16
    b = make_batch(orc, S, H, W, N, seed0=4200, dtype="f32", P=S, G=S)
    _, g0, _ = _run(b, torch.float32, False)
    _, g1, _ = _run(b, torch.float32, True)
    for k in ("dB", "dC"):
        assert rel_error(g1[k].reshape(-1), g0[k].reshape(-1)) <= 2e-6, k
    ref = oracle_bwd(orc, b, "f64")
    for k in ("dB", "dC"):
        assert rel_error(g1[k].reshape(-1), np.asarray(ref[k]).reshape(-1)) <= 1e-4, k


@pytest.mark.gpu
@pytest.mark.parametrize("misalign", ["outputs", "workspace"])
def test_group_red_unaligned_destinations(orc, misalign):
    """With the flag set, dB / dC at an odd element offset must not take
    16-byte vector stores (the planner then runs the scalar-store kernels
    through the workspace path); a workspace off 16-byte alignment is refused
    (SCAN2D_EINVAL, include/scan2d_cuda.h) instead of faulting."""
    import ctypes as C

    from paper_2412_00678_b200 import _native as nat
    from paper_2412_00678_b200.api import Scan2dOp

    S, H, W, N, G = 6, 20, 40, 16, 3
    b = make_batch(orc, S, H, W, N, seed0=4300, dtype="f32", P=S, G=G)
    (x, z, B, C_, A, D, bias), dy = batch_to_torch(b, device="cuda")
    op = Scan2dOp(S, H, W, N, bc_group=G, device="cuda", group_red=True)
    op.forward(x, z, B, C_, A, D, bias)
    shapes = [(S, H, W), (S, H, W), (S, N), (S // G, H, W, N), (S // G, H, W, N), (S,), (S,)]
    off = 1 if misalign == "outputs" else 0
    outs = [torch.full((int(np.prod(s)) + off,), float("nan"), device="cuda")[off:].view(s) for s in shapes]
    wsb = op.wsb_bytes
    wbuf = torch.empty(wsb + 64, dtype=torch.uint8, device="cuda")
    ws = wbuf[4:] if misalign == "workspace" else wbuf
    p = lambda t: C.c_void_p(t.data_ptr())
    rc = nat.lib.scan2d_backward(C.byref(op.desc), p(x), p(z), p(B), p(C_), p(A), p(D), p(bias), p(op.residual),
                                 p(dy), *[p(o) for o in outs], p(ws), wsb,
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if misalign == "workspace":  # documented requirement: 16-byte aligned workspace / residual
        assert rc == nat.EINVAL
        return
    assert rc == nat.OK, nat.status_string(rc)
    torch.cuda.synchronize()
    ref = oracle_bwd(orc, b, "f64")
    for k, name in enumerate(NAMES):
        assert rel_error(outs[k].cpu().numpy().reshape(-1), np.asarray(ref[name]).reshape(-1)) <= 1e-4, name
