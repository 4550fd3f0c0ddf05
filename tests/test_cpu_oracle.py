"""CPU-only tests: the oracle pinned against the reference (golden vectors and,
where it was built, the reference library itself), the C-ABI library's
exports and host-side validation, and the reference's own doctest suite.
No GPU is touched here."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle_lib import REF_SO, Oracle, RefLib, rel_error

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")
HEADER = os.path.join(REPO, "include", "scan2d_cuda.h")
LIB = os.path.join(REPO, "paper_2412_00678_b200", "lib", "libscan2d_cuda.so")
SHIM = os.path.join(REPO, "paper_2412_00678_b200", "lib", "libscan2d_engine_cuda.so")

FWD_CASES = [(11, 7, 4, (64,), 42), (6, 9, 3, (1,), 43), (8, 8, 2, (3,), 44), (13, 10, 5, (1, 2, 3, 8, 13), 45),
             (33, 29, 6, (8,), 48), (23, 17, 3, (8,), 1000 + 23 * 31 + 17)]
BWD_CASES = [(5, 6, 3, 2, 60), (7, 4, 2, 3, 62), (5, 4, 3, 3, 0), (4, 5, 2, 6, 7), (17, 13, 4, 4, 63),
             (16, 16, 16, 16, 1000)]


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


# ------------------------------------------------------ oracle vs golden


@pytest.mark.parametrize("h,w,n,tiles,seed", FWD_CASES)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_oracle_forward_matches_golden(orc, golden, h, w, n, tiles, seed, dt):
    key = f"fwd_{h}x{w}_n{n}_s{seed}_{dt}"
    inst = orc.random_instance(h, w, n, seed, dt)
    # the generator restatement reproduces the reference fixtures bit for bit
    assert np.array_equal(inst.x, golden[key + "_x"])
    assert np.array_equal(inst.B, golden[key + "_B"])
    y = orc.fwd(inst, dt)
    for t in tiles:
        # tiled reference engine == sequential oracle bit for bit (same op order per element)
        assert np.array_equal(y, golden[f"{key}_t{t}_y"]), f"T={t}"
        ph, pv = orc.carries(inst, t, dt)
        assert np.array_equal(ph, golden[f"{key}_t{t}_ph"])
        assert np.array_equal(pv, golden[f"{key}_t{t}_pv"])


@pytest.mark.parametrize("h,w,n,t,seed", BWD_CASES)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_oracle_backward_matches_golden(orc, golden, h, w, n, t, seed, dt):
    key = f"bwd_{h}x{w}_n{n}_s{seed}_t{t}_{dt}"
    inst = orc.random_instance(h, w, n, seed, dt)
    dy = orc.fill_normal(seed ^ 0x5EED, h * w, "f64").astype(np.float64 if dt == "f64" else np.float32)
    g = orc.bwd(inst, dy, dt)
    for k in ("dx", "dz", "dB", "dC"):  # per-element chain rule: identical operations
        assert np.array_equal(g[k], golden[f"{key}_{k}"]), k
    # scalar groups: the reference sums tile-major (engine.cpp:404-408), the
    # oracle row-major -- equal up to summation order
    tol = 1e-13 if dt == "f64" else 2e-5
    for k in ("dA", "dD", "dbias"):
        assert rel_error(g[k], golden[f"{key}_{k}"]) <= tol, k


def test_oracle_config1_matches_golden(orc, golden):
    """BASELINE.json configs[0]: 64 scans, 16x16, N=16, fp32."""
    ys = golden["cfg1_y_f32"]
    for s in range(64):
        inst = orc.random_instance(16, 16, 16, 1000 + s, "f32")
        assert np.array_equal(orc.fwd(inst, "f32"), ys[s])


def test_oracle_fast_expf_known_values(orc):
    L = orc.lib
    assert L.orc_fast_expf(0.0) == 1.0
    assert L.orc_fast_expf(-100.0) == 0.0  # flush below -87.33654 (math.hpp:44-45)
    xs = np.linspace(-87, 88, 2001, dtype=np.float32)
    got = np.array([L.orc_fast_expf(float(v)) for v in xs], np.float64)
    assert np.max(np.abs(got - np.exp(xs.astype(np.float64))) / np.exp(xs.astype(np.float64))) < 5e-7


def test_oracle_closed_form(orc):
    """Constant Abar = a, Bbar x = b: h(i,j) = b (1-a^(i+1))(1-a^(j+1)) / (1-a)^2
    (reference.cpp:116-127, test_reference.cpp:171-195)."""
    from oracle_lib import Instance

    h, w = 9, 11
    a = 0.5
    inst = Instance(h, w, 1, np.ones(h * w), np.full(h * w, np.log(np.e - 1.0)), np.full(h * w, 0.75),
                    np.ones(h * w), np.array([np.log(a)]), 0.0, 0.0)
    y = orc.fwd(inst, "f64").reshape(h, w)
    i = np.arange(h)[:, None]
    j = np.arange(w)[None, :]
    expect = 0.75 * (1 - a ** (i + 1)) * (1 - a ** (j + 1)) / (1 - a) ** 2
    assert rel_error(y, expect) <= 1e-14


def test_oracle_gradcheck_golden(golden):
    """The reference's own FD gradcheck numbers pass its tolerances (test_backward.cpp:39-46)."""
    g = golden["gradcheck_5x4_n3_s0_t3"]
    assert np.all(g[:, 0] <= 1e-6) and np.all(g[:, 1] <= 1e-9)


# ------------------------------------------------- oracle vs reference lib

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built here")


@needs_ref
def test_oracle_vs_reference_random(orc):
    ref = RefLib()
    rng = np.random.default_rng(5)
    for _ in range(20):
        h, w, n = (int(v) for v in rng.integers(1, 20, 3))
        t = int(rng.choice([1, 2, 3, 8, 64]))
        seed = int(rng.integers(0, 2**31))
        for dt in ("f64", "f32"):
            a = orc.random_instance(h, w, n, seed, dt)
            y_ref, ph_ref, pv_ref = ref.tiled_fwd(ref.random_instance(h, w, n, seed, dt), t, dt)
            assert np.array_equal(orc.fwd(a, dt), y_ref)
            ph, pv = orc.carries(a, t, dt)
            assert np.array_equal(ph, ph_ref) and np.array_equal(pv, pv_ref)
            dy = orc.fill_normal(seed ^ 0x5EED, h * w, dt)
            g = orc.bwd(a, dy, dt)
            gr = ref.tiled_bwd(ref.random_instance(h, w, n, seed, dt), 10**6, dy, dt)  # one tile
            for k in ("dx", "dz", "dB", "dC", "dA", "dD", "dbias"):
                assert np.array_equal(np.asarray(g[k]).ravel(), np.asarray(gr[k]).ravel()), k


@needs_ref
def test_oracle_fast_expf_bitexact_vs_reference(orc):
    ref = RefLib()
    for v in np.linspace(-90, 89, 5001, dtype=np.float32):
        assert orc.lib.orc_fast_expf(float(v)) == ref.lib.ref_fast_expf(float(v))


@pytest.mark.skipif(not os.path.exists(os.path.join(REPO, "oracle", "_ref", "ref_tests")),
                    reason="reference doctest suite not built")
def test_reference_suite_against_reference_engine():
    """The reference's own unit tests (engine, backward, reference, block_scan,
    memsim; T2DM I/O is out of scope) pass under our doctest-compatible harness."""
    r = subprocess.run([os.path.join(REPO, "oracle", "_ref", "ref_tests")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


# ------------------------------------------------------------- the C ABI


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(scan2d_[a-z0-9_]+)\s*\(", txt)))


def test_capi_exports_every_header_symbol():
    assert os.path.exists(LIB), "build the CUDA library first (__graft_entry__.build())"
    lib = C.CDLL(LIB)
    names = header_functions()
    assert len(names) >= 13
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/scan2d_cuda.h but not exported"
    from paper_2412_00678_b200 import _native

    assert sorted(_native.EXPORTED_SYMBOLS) == names


def test_t2dm_exports_every_header_symbol():
    lib = C.CDLL(LIB)
    txt = re.sub(r"/\*.*?\*/", "", open(os.path.join(os.path.dirname(HEADER), "scan2d_t2dm.h")).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(scan2d_t2dm_[a-z0-9_]+)\s*\(", txt)))
    assert len(names) == 7
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/scan2d_t2dm.h but not exported"


def test_capi_descriptor_validation():
    from paper_2412_00678_b200 import _native as nat

    lib = nat.lib
    ok = nat.make_desc(4, 8, 9, 16)
    assert lib.scan2d_check_desc(C.byref(ok)) == nat.OK
    bad = [nat.make_desc(0, 8, 9, 16), nat.make_desc(4, 0, 9, 16), nat.make_desc(4, 8, 0, 16),
           nat.make_desc(4, 8, 9, 0), nat.make_desc(4, 8, 9, 2049), nat.make_desc(4, 8, 9, 16, tile=0),
           nat.make_desc(4, 8, 9, 16, params_period=3), nat.make_desc(4, 8, 9, 16, bc_group=3),
           nat.make_desc(4, 8, 9, 16, dtype=7)]
    for d in bad:
        assert lib.scan2d_check_desc(C.byref(d)) == nat.EINVAL
        # entry points reject before touching the device
        assert lib.scan2d_forward(C.byref(d), *([None] * 12), 0, None) == nat.EINVAL
        assert lib.scan2d_backward(C.byref(d), *([None] * 17), 0, None) == nat.EINVAL
    assert lib.scan2d_backward(C.byref(ok), *([None] * 17), 0, None) == nat.ESTALE
    assert nat.status_string(nat.ESTALE).startswith("stale")
    assert lib.scan2d_version() >= 1


def test_capi_sizes_and_plans():
    from paper_2412_00678_b200 import _native as nat

    lib = nat.lib
    for S, H, W, N in [(64, 16, 16, 16), (128, 200, 200, 16), (12288, 56, 56, 1), (256, 1024, 1024, 16),
                       (49152, 7, 7, 1), (5, 9, 300, 3), (2, 3, 5, 32)]:
        d = nat.make_desc(S, H, W, N)
        assert lib.scan2d_workspace_bytes(C.byref(d), nat.OP_FWD) > 0
        assert lib.scan2d_workspace_bytes(C.byref(d), nat.OP_BWD) > 0
        assert lib.scan2d_residual_bytes(C.byref(d)) > 0
        f = nat.plan_info(d, nat.OP_FWD)
        b = nat.plan_info(d, nat.OP_BWD)
        for p in (f, b):
            assert p["smem_bytes"] <= 200 * 1024
            assert p["warps_total"] >= 1
            # every column of every scan is covered
            assert p["cols_per_warp"] * p["warps_per_scan"] >= W
            assert p["scans_per_warp"] * p["warps_total"] >= S * p["warps_per_scan"] // max(p["warps_per_scan"], 1)


@pytest.mark.skipif(not os.path.exists(SHIM), reason="engine shim not built (needs the reference headers)")
def test_engine_shim_exports_reference_api():
    out = subprocess.run(["nm", "-DC", SHIM], capture_output=True, text=True).stdout
    for sym in ("scan2d::tiled_scan_2d_forward<float>", "scan2d::tiled_scan_2d_forward<double>",
                "scan2d::tiled_scan_2d_backward<float>", "scan2d::tiled_scan_2d_backward<double>",
                "scan2d::naive_scan_2d<double>", "scan2d::block_scan_1d_forward<float>"):
        assert sym in out, sym


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: importing the binding without its shared object raises."""
    import subprocess
    import sys as _sys

    code = "import paper_2412_00678_b200._native"
    env = dict(os.environ, SCAN2D_LIB_PATH=str(tmp_path / "missing.so"))
    p = subprocess.run([_sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True, text=True)
    assert p.returncode != 0
    assert "missing.so" in p.stderr or "OSError" in p.stderr
