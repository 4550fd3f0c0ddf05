"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Mirrors the reference's engine/backward acceptance cases
(proj/tests/test_engine.cpp, proj/tests/test_backward.cpp) on the batched
layout, plus the BASELINE.json shapes.  Gates:
  fp64: normwise rel_error <= 1e-12 (y) / 1e-10 (grads) vs the fp64 oracle
  fp32: normwise rel_error <= 1e-4 vs the fp64 oracle on the same fp32 inputs
        (north_star tolerance), and <= 1e-5 vs the fp32 oracle for y
        (test_engine.cpp:69).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle_lib import Oracle, elem_stats, rel_error
from scan_cases import batch_to_torch, make_batch, oracle_bwd, oracle_fwd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

F32_GATE = 1e-4
F64_Y_GATE = 1e-12
F64_G_GATE = 1e-10


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def s2d():
    import paper_2412_00678_b200 as m

    return m


def run_fwd(s2d, b, dtype, tile=16, carries=False, save=True):
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b, dtype=dtype)
    res = s2d.tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=tile, carries=carries, save_residuals=save)
    torch.cuda.synchronize()
    return res, dy


def grads_np(g):
    return dict(dx=g.dx.cpu().numpy(), dz=g.dz_raw.cpu().numpy(), dA=g.da.cpu().numpy(),
                dB=g.db.cpu().numpy(), dC=g.dc.cpu().numpy(), dD=g.dd.cpu().numpy(),
                dbias=g.dbias.cpu().numpy())


def check_grads(got, ref, gate, label):
    for k in ("dx", "dz", "dA", "dB", "dC", "dD", "dbias"):
        e = rel_error(got[k], ref[k])
        assert e <= gate, f"{label}: {k} rel_error {e:.3e} > {gate:.0e}"


# ------------------------------------------------------------------ forward


@pytest.mark.parametrize("H,W,N,T,seed", [(11, 7, 4, 64, 42), (6, 9, 3, 1, 43), (8, 8, 2, 3, 44),
                                          (13, 10, 5, 8, 45), (33, 29, 6, 8, 48)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_forward_reference_cases(orc, s2d, H, W, N, T, seed, dtype):
    """test_engine.cpp:12-44 shapes, single scan."""
    b = make_batch(orc, 1, H, W, N, seed0=seed, dtype=dtype)
    res, _ = run_fwd(s2d, b, torch.float64 if dtype == "f64" else torch.float32, tile=T)
    y = res.y.cpu().numpy()
    y64 = oracle_fwd(orc, b, "f64")
    if dtype == "f64":
        assert rel_error(y, y64) <= F64_Y_GATE
    else:
        assert rel_error(y, y64) <= F32_GATE
        assert rel_error(y, oracle_fwd(orc, b, "f32")) <= 1e-5


def test_forward_random_trials(orc, s2d):
    """test_engine.cpp:46-73: 30 random shapes (H, W <= 24, N <= 8, T in {1,2,3,8,64}),
    drawn from the same meta-generator Rng(46) as the reference."""
    meta = _MetaRng(orc, 46)
    for trial in range(30):
        h = meta.uniform_int(1, 24)
        w = meta.uniform_int(1, 24)
        n = meta.uniform_int(1, 8)
        t = [1, 2, 3, 8, 64][meta.uniform_int(0, 4)]
        seed = meta.next_u64()
        for dtype, gate in (("f64", F64_Y_GATE), ("f32", F32_GATE)):
            b = make_batch(orc, 1, h, w, n, seed0=seed, dtype=dtype)
            res, _ = run_fwd(s2d, b, torch.float64 if dtype == "f64" else torch.float32, tile=t)
            e = rel_error(res.y.cpu().numpy(), oracle_fwd(orc, b, "f64"))
            assert e <= gate, f"trial {trial} {dtype} {h}x{w} n={n} t={t}: {e:.3e}"


class _MetaRng:
    """Rng (rng.hpp) driven through the oracle library."""

    def __init__(self, orc, seed):
        import ctypes as C

        self.C = C
        self.lib = orc.lib
        self.lib.orc_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        self.lib.orc_rng_next.argtypes = [C.c_void_p]
        self.lib.orc_rng_next.restype = C.c_uint64
        self.lib.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        self.lib.orc_rng_uniform_int.restype = C.c_int
        self.buf = C.create_string_buffer(32)
        self.lib.orc_rng_init(self.buf, C.c_uint64(seed))

    def uniform_int(self, lo, hi):
        return self.lib.orc_rng_uniform_int(self.buf, lo, hi)

    def next_u64(self):
        return self.lib.orc_rng_next(self.buf)


@pytest.mark.parametrize("H,W,N,T", [(9, 9, 2, 4), (16, 16, 16, 16), (23, 17, 3, 8), (7, 7, 2, 16),
                                     (40, 300, 16, 16), (7, 9, 260, 4)])
def test_forward_carries(orc, s2d, H, W, N, T):
    """CarryState ph / pv (engine.hpp:29-46) including edge pass-through slots."""
    b = make_batch(orc, 2, H, W, N, seed0=7, dtype="f64")
    res, _ = run_fwd(s2d, b, torch.float64, tile=T, carries=True)
    for s in range(2):
        from oracle_lib import Instance

        inst = Instance(H, W, N, b.x[s].ravel(), b.z[s].ravel(), b.B[s].ravel(), b.C[s].ravel(), b.A[s],
                        float(b.D[s]), float(b.bias[s]))
        ph, pv = orc.carries(inst, T, "f64")
        assert rel_error(res.ph[s].cpu().numpy().ravel(), ph) <= 1e-12
        assert rel_error(res.pv[s].cpu().numpy().ravel(), pv) <= 1e-12


def test_forward_zero_input(orc, s2d):
    """test_engine.cpp:28-34: x = 0 => y == 0 exactly."""
    b = make_batch(orc, 3, 8, 8, 2, seed0=44, dtype="f64")
    b.x[:] = 0
    res, _ = run_fwd(s2d, b, torch.float64, tile=3)
    assert np.all(res.y.cpu().numpy() == 0.0)


@pytest.mark.parametrize("S,H,W,N", [(64, 16, 16, 16),    # config 1 (BASELINE.json configs[0])
                                     (40, 56, 56, 1), (24, 28, 28, 1), (48, 14, 14, 1), (64, 7, 7, 1),
                                     (6, 200, 200, 16), (3, 24, 1024, 16), (4, 33, 700, 1), (5, 9, 300, 3)])
def test_forward_batched_shapes(orc, s2d, S, H, W, N):
    b = make_batch(orc, S, H, W, N, seed0=1000, dtype="f32")
    res, _ = run_fwd(s2d, b, torch.float32)
    y = res.y.cpu().numpy()
    y64 = oracle_fwd(orc, b, "f64")
    e = rel_error(y, y64)
    st = elem_stats(y, y64)
    assert e <= F32_GATE, f"{S}x{H}x{W} N={N}: rel {e:.3e} stats {st}"


def test_forward_shared_params_and_bc(orc, s2d):
    """params per channel (P < S) and B/C shared across G scans (model.cpp:150-193)."""
    b = make_batch(orc, 12, 20, 37, 8, seed0=5, dtype="f64", P=4, G=3)
    res, _ = run_fwd(s2d, b, torch.float64)
    assert rel_error(res.y.cpu().numpy(), oracle_fwd(orc, b, "f64")) <= F64_Y_GATE


def test_forward_deterministic(orc, s2d):
    b = make_batch(orc, 8, 45, 130, 16, seed0=48, dtype="f32")
    r1, _ = run_fwd(s2d, b, torch.float32, carries=True)
    r2, _ = run_fwd(s2d, b, torch.float32, carries=True)
    assert torch.equal(r1.y, r2.y) and torch.equal(r1.ph, r2.ph) and torch.equal(r1.pv, r2.pv)


# ----------------------------------------------------------------- backward


@pytest.mark.parametrize("S,H,W,N,dtype", [(1, 5, 4, 3, "f64"), (1, 4, 5, 2, "f64"), (2, 17, 13, 4, "f64"),
                                           (3, 19, 23, 8, "f64"), (2, 9, 300, 3, "f64"), (2, 12, 1024, 16, "f64"),
                                           (64, 16, 16, 16, "f32"), (16, 56, 56, 1, "f32"), (32, 7, 7, 1, "f32"),
                                           (2, 200, 200, 16, "f32"), (2, 21, 700, 1, "f32")])
def test_backward_vs_oracle(orc, s2d, S, H, W, N, dtype):
    b = make_batch(orc, S, H, W, N, seed0=60, dtype=dtype)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    res, dy = run_fwd(s2d, b, tdt)
    g = s2d.tiled_scan_2d_backward(res.saved, dy)
    torch.cuda.synchronize()
    ref = oracle_bwd(orc, b, "f64")
    check_grads(grads_np(g), ref, F64_G_GATE if dtype == "f64" else F32_GATE, f"{S}x{H}x{W} N={N} {dtype}")


def test_backward_shared_params_and_bc(orc, s2d):
    b = make_batch(orc, 12, 20, 37, 8, seed0=5, dtype="f64", P=4, G=3)
    res, dy = run_fwd(s2d, b, torch.float64)
    g = s2d.tiled_scan_2d_backward(res.saved, dy)
    check_grads(grads_np(g), oracle_bwd(orc, b, "f64"), F64_G_GATE, "shared P=4 G=3")


def test_backward_zero_dy(orc, s2d):
    """test_backward.cpp:11-23: dy = 0 => every gradient exactly 0."""
    b = make_batch(orc, 2, 5, 6, 3, seed0=60, dtype="f64")
    res, dy = run_fwd(s2d, b, torch.float64, tile=2)
    g = s2d.tiled_scan_2d_backward(res.saved, torch.zeros_like(dy))
    for v in grads_np(g).values():
        assert np.all(v == 0.0)


def test_backward_dD_identity(orc, s2d):
    """test_backward.cpp:25-37: dD == sum dy * x."""
    b = make_batch(orc, 1, 7, 4, 2, seed0=62, dtype="f64")
    res, dy = run_fwd(s2d, b, torch.float64, tile=3)
    g = s2d.tiled_scan_2d_backward(res.saved, dy)
    expect = float((b.dy * b.x).sum())
    assert abs(float(g.dd[0]) - expect) <= 1e-12 * (1 + abs(expect))


def test_backward_deterministic(orc, s2d):
    """test_backward.cpp:56-74: bit-identical across runs."""
    b = make_batch(orc, 4, 33, 640, 16, seed0=63, dtype="f32")
    res, dy = run_fwd(s2d, b, torch.float32)
    g1 = grads_np(s2d.tiled_scan_2d_backward(res.saved, dy))
    g2 = grads_np(s2d.tiled_scan_2d_backward(res.saved, dy))
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k


def test_error_paths(orc, s2d):
    """test_engine.cpp:125-134 / test_backward.cpp:76-92 error types."""
    b = make_batch(orc, 1, 4, 4, 2, seed0=51, dtype="f64")
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b)
    with pytest.raises(ValueError):
        s2d.tiled_scan_2d_forward(x, z[:, :, :3].contiguous(), B, C, A, D, bias)
    with pytest.raises(ValueError):
        s2d.tiled_scan_2d_forward(x, z, B, C, A[:, :1].contiguous(), D, bias)
    with pytest.raises(ValueError):
        s2d.tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=0)
    with pytest.raises(RuntimeError):
        s2d.tiled_scan_2d_backward(s2d.SavedForward(), dy)
    res = s2d.tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=2)
    with pytest.raises(ValueError):
        s2d.tiled_scan_2d_backward(res.saved, torch.zeros((1, 4, 5), dtype=dy.dtype, device=dy.device))
    inf = s2d.tiled_scan_2d_forward(x, z, B, C, A, D, bias, tile=2, save_residuals=False)
    assert not inf.saved.valid
    with pytest.raises(RuntimeError):
        s2d.tiled_scan_2d_backward(inf.saved, dy)


def test_autograd_function(orc, s2d):
    b = make_batch(orc, 3, 10, 12, 4, seed0=9, dtype="f64")
    (x, z, B, C, A, D, bias), dy = batch_to_torch(b)
    ins = [t.clone().requires_grad_(True) for t in (x, z, B, C, A, D, bias)]
    y = s2d.scan2d(*ins)
    (y * dy).sum().backward()
    ref = oracle_bwd(orc, b, "f64")
    got = dict(dx=ins[0].grad, dz=ins[1].grad, dB=ins[2].grad, dC=ins[3].grad, dA=ins[4].grad,
               dD=ins[5].grad, dbias=ins[6].grad)
    check_grads({k: v.cpu().numpy() for k, v in got.items()}, ref, F64_G_GATE, "autograd")


def test_closed_form_large_grid(s2d):
    """Constant Abar = a, Bbar x = b: h(i,j) = b (1-a^(i+1))/(1-a) (1-a^(j+1))/(1-a)
    (reference.cpp:116-127) -- a size-independent check at 1024 x 1024."""
    H = W = 1024
    N = 1
    a_target = 0.9
    dev = "cuda"
    # delta = softplus(z + bias) = 1 (z = log(e - 1)), A = log(a): Abar = a; B x = b / delta
    zval = float(np.log(np.e - 1.0))
    x = torch.ones((1, H, W), dtype=torch.float64, device=dev)
    z = torch.full((1, H, W), zval, dtype=torch.float64, device=dev)
    B = torch.full((1, H, W, N), 0.5, dtype=torch.float64, device=dev)
    C = torch.ones((1, H, W, N), dtype=torch.float64, device=dev)
    A = torch.full((1, N), float(np.log(a_target)), dtype=torch.float64, device=dev)
    D = torch.zeros((1,), dtype=torch.float64, device=dev)
    bias = torch.zeros((1,), dtype=torch.float64, device=dev)
    y = s2d.tiled_scan_2d_forward(x, z, B, C, A, D, bias, save_residuals=False).y[0].cpu().numpy()
    i = np.arange(H)[:, None]
    j = np.arange(W)[None, :]
    geo = lambda k: (1 - a_target ** (k + 1)) / (1 - a_target)
    expect = 0.5 * geo(i) * geo(j)
    assert rel_error(y, expect) <= 1e-12


# ------------------------------------------------- reference golden vectors

GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)),
                                    "golden", "reference_golden.npz")
FWD_GOLD = [(11, 7, 4, (64,), 42), (6, 9, 3, (1,), 43), (8, 8, 2, (3,), 44), (13, 10, 5, (1, 2, 3, 8, 13), 45),
            (33, 29, 6, (8,), 48), (23, 17, 3, (8,), 1000 + 23 * 31 + 17)]
BWD_GOLD = [(5, 6, 3, 2, 60), (7, 4, 2, 3, 62), (5, 4, 3, 3, 0), (4, 5, 2, 6, 7), (17, 13, 4, 4, 63),
            (16, 16, 16, 16, 1000)]


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_forward_vs_reference_golden(orc, s2d, dt):
    """y and the CarryState against numbers produced by the reference library itself."""
    gold = np.load(GOLDEN)
    gate = F64_Y_GATE if dt == "f64" else 1e-5
    tdt = torch.float64 if dt == "f64" else torch.float32
    for h, w, n, tiles, seed in FWD_GOLD:
        key = f"fwd_{h}x{w}_n{n}_s{seed}_{dt}"
        b = make_batch(orc, 1, h, w, n, seed0=seed, dtype=dt)
        assert np.array_equal(b.x.ravel(), gold[key + "_x"])
        for t in tiles:
            res, _ = run_fwd(s2d, b, tdt, tile=t, carries=True)
            assert rel_error(res.y.cpu().numpy(), gold[f"{key}_t{t}_y"]) <= gate, (key, t)
            assert rel_error(res.ph.cpu().numpy(), gold[f"{key}_t{t}_ph"]) <= gate, (key, t)
            assert rel_error(res.pv.cpu().numpy(), gold[f"{key}_t{t}_pv"]) <= gate, (key, t)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_backward_vs_reference_golden(orc, s2d, dt):
    gold = np.load(GOLDEN)
    tdt = torch.float64 if dt == "f64" else torch.float32
    for h, w, n, t, seed in BWD_GOLD:
        key = f"bwd_{h}x{w}_n{n}_s{seed}_t{t}_{dt}"
        b = make_batch(orc, 1, h, w, n, seed0=seed, dtype=dt)
        res, dy = run_fwd(s2d, b, tdt, tile=t)
        g = grads_np(s2d.tiled_scan_2d_backward(res.saved, dy))
        for k in ("dx", "dz", "dA", "dB", "dC", "dD", "dbias"):
            e = rel_error(g[k], gold[f"{key}_{k}"])
            assert e <= (F64_G_GATE if dt == "f64" else F32_GATE), (key, k, e)


def test_config1_vs_reference_golden(orc, s2d):
    """BASELINE.json configs[0] (64 scans, 16x16, N=16, fp32): the batched GPU
    forward against the reference engine's outputs, scan by scan."""
    gold = np.load(GOLDEN)["cfg1_y_f32"]
    b = make_batch(orc, 64, 16, 16, 16, seed0=1000, dtype="f32")
    res, _ = run_fwd(s2d, b, torch.float32)
    y = res.y.cpu().numpy().reshape(64, -1)
    for s in range(64):
        assert rel_error(y[s], gold[s]) <= 1e-5


def test_reference_suite_against_cuda_engine():
    """The reference's own doctest suites (engine, backward, memsim, reference,
    block_scan) linked against the CUDA engine shim instead of engine.cpp."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "ref_tests_cuda")
    if not os.path.exists(exe):
        pytest.skip("ref_tests_cuda not built (needs the reference sources at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert " 0 failed" in r.stdout


# ------------------------------------------------------------- comparators


def _variant(s2d, b, variant, dtype):
    import ctypes as C

    from paper_2412_00678_b200 import _native as nat

    (x, z, B, Cc, A, D, bias), _ = batch_to_torch(b, dtype=dtype)
    desc = nat.make_desc(b.S, b.H, b.W, b.N, params_period=b.P, bc_group=b.G,
                         dtype=nat.F64 if dtype == torch.float64 else nat.F32)
    y = torch.empty_like(x)
    wsb = nat.lib.scan2d_comparator_workspace_bytes(C.byref(desc), variant)
    ws = torch.empty(wsb, dtype=torch.uint8, device=x.device)
    p = lambda t: C.c_void_p(t.data_ptr())
    rc = nat.lib.scan2d_forward_variant(C.byref(desc), variant, p(x), p(z), p(B), p(Cc), p(A), p(D), p(bias), p(y),
                                        p(ws), wsb, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == nat.OK
    torch.cuda.synchronize()
    return y.cpu().numpy()


def test_naive_comparator_vs_oracle(orc, s2d):
    from paper_2412_00678_b200 import _native as nat

    b = make_batch(orc, 3, 13, 17, 5, seed0=71, dtype="f64")
    assert rel_error(_variant(s2d, b, nat.VARIANT_NAIVE, torch.float64), oracle_fwd(orc, b, "f64")) <= F64_Y_GATE


@pytest.mark.parametrize("S,H,W,N,dt", [(2, 5, 8, 3, "f64"), (2, 30, 40, 16, "f64"), (3, 14, 14, 16, "f64"),
                                         (2, 23, 29, 4, "f64"), (2, 56, 56, 16, "f32"), (1, 1, 1, 1, "f64"),
                                         (2, 7, 73, 8, "f32")])
def test_flat1d_comparator_vs_sequential(orc, s2d, S, H, W, N, dt):
    """block_scan_1d_forward == scan_1d_sequential on the row-major flattening
    (test_engine.cpp:75-82); N in {1, 2, 4, 8, 16} runs the block-scan kernel
    (chunk boundaries at 512 elements), other N the sequential one."""
    from paper_2412_00678_b200 import _native as nat

    b = make_batch(orc, S, H, W, N, seed0=47, dtype=dt)
    y = _variant(s2d, b, nat.VARIANT_FLAT1D, torch.float64 if dt == "f64" else torch.float32)
    gate = 1e-12 if dt == "f64" else 1e-4
    for s in range(b.S):
        L = b.H * b.W
        x, z = b.x[s].ravel(), b.z[s].ravel()
        B, Cc = b.B[s].reshape(L, b.N), b.C[s].reshape(L, b.N)
        x, z, B, Cc = [np.asarray(v, np.float64) for v in (x, z, B, Cc)]
        A, D, bias = np.asarray(b.A[s], np.float64), float(b.D[s]), float(b.bias[s])
        delta = np.where(z + bias > 20, z + bias, np.log1p(np.exp(z + bias)))
        h = np.zeros(b.N)
        ref = np.empty(L)
        for k in range(L):
            h = np.exp(delta[k] * A) * h + delta[k] * B[k] * x[k]
            ref[k] = (Cc[k] * h).sum() + D * x[k]
        assert rel_error(y[s].ravel(), ref) <= gate
