"""scan2d_cli: usage errors on the CPU;
scan / verify / gradcheck / bench on the GPU, with the scan's T2DM output
checked against the fp64 oracle on the same inputs."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle_lib import Oracle, rel_error
from scan_cases import make_batch, oracle_fwd

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_2412_00678_b200", "lib", "scan2d_cli")


def run(*args, check_rc=None):
    p = subprocess.run([CLI, *[str(a) for a in args]], capture_output=True, text=True, timeout=600)
    if check_rc is not None:
        assert p.returncode == check_rc, (p.returncode, p.stdout, p.stderr)
    return p


def lines(p):
    return [json.loads(v) for v in p.stdout.splitlines() if v.strip()]


@pytest.mark.skipif(not os.path.exists(CLI), reason="scan2d_cli not built")
@pytest.mark.parametrize("args", [[], ["bogus"], ["verify"], ["bench", "--height"], ["scan", "--nope", "1"],
                                  ["bench", "--height", "x"], ["verify", "--sizes", "3y4"]])
def test_usage_errors_exit_2(args):
    p = run(*args)
    assert p.returncode == 2 and "usage" in p.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,N", [("f32", 16), ("f64", 4), ("f32", 1), ("f32", 5)])
def test_verify(dtype, N):
    p = run("verify", "--sizes", "16x16,14x14,56x56,3x200,1x1", "--seeds", "0,1", "--dtype", dtype, "--state-dim", N,
            check_rc=0)
    out = lines(p)
    assert len(out) == 10 and all(o["pass"] and o["tile_invariant"] for o in out), out


@pytest.mark.gpu
def test_gradcheck():
    # the reference gradcheck test case (test_backward.cpp:40): 5 x 4, N = 3, every component
    out = lines(run("gradcheck", "--height", 5, "--width", 4, "--state-dim", 3, "--seed", 0, check_rc=0))[0]
    assert out["pass"] and set(out["groups"]) == {"dx", "dz_raw", "da", "db", "dc", "dd", "dbias"}


@pytest.mark.gpu
@pytest.mark.parametrize("S,H,W,N,variant", [(1, 12, 20, 16, "tiled2d"), (3, 9, 30, 8, "tiled2d"),
                                             (2, 7, 9, 4, "naive2d"), (2, 6, 11, 16, "seq1d")])
def test_scan_t2dm_round_trip(tmp_path, S, H, W, N, variant):
    from paper_2412_00678_b200 import t2dm

    orc = Oracle()
    b = make_batch(orc, S, H, W, N, seed0=900, dtype="f64")
    f = lambda name, a: (t2dm.write(tmp_path / name, np.ascontiguousarray(a)), str(tmp_path / name))[1]  # noqa: E731
    x = b.x[0] if S == 1 else b.x  # [H,W] (T2DM v1) for one scan, [S,H,W] (v2) for a batch
    args = ["scan", "--input", f("x.t2dm", x), "--output", tmp_path / "y.t2dm", "--variant", variant,
            "--state-dim", N, "--dtype", "f64", "--z", f("z.t2dm", b.z), "--b", f("b.t2dm", b.B),
            "--c", f("c.t2dm", b.C), "--a", f("a.t2dm", b.A), "--dskip", f("d.t2dm", b.D),
            "--bias", f("bias.t2dm", b.bias)]
    out = lines(run(*args, check_rc=0))[0]
    assert out["variant"] == variant and out["scans"] == S
    y = t2dm.read(tmp_path / "y.t2dm")
    assert y.shape == ((H, W) if S == 1 else (S, H, W))
    if variant == "seq1d":  # the flattened 1D scan is a different operator: compare shape only
        return
    assert rel_error(y.reshape(S, H, W), oracle_fwd(orc, b, "f64")) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("variant,extra", [("tiled2d", ["--backward"]), ("tiled2d", []), ("naive2d", []),
                                           ("seq1d", [])])
def test_bench_result(variant, extra):
    out = lines(run("bench", "--variant", variant, "--height", 56, "--width", 56, "--state-dim", 16, "--batch", 8,
                    "--reps", 5, "--warmup", 2, *extra, check_rc=0))[0]
    for k in ("variant", "height", "width", "state_dim", "tile", "dtype", "repetitions", "wall_time_per_rep_s",
              "throughput_maps_per_s", "flops", "mem_report"):
        assert k in out
    assert out["throughput_maps_per_s"] > 0
    assert abs(out["throughput_maps_per_s"] * out["wall_time_per_rep_s"] - out["batch"]) < 1e-6 * out["batch"]
